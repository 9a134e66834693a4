// Combinatorial ranks of monomials (grevlex rank-bitmap dictionary).
//
// For grevlex and batch degree <= D every monomial m has a rank
//   rank(m) = C(n+d-1, n) + sum_{i=n-1..1} [s_i > e_i] C(s_i - e_i - 1 + i, i),
//   d = deg m, s_{n-1} = d, s_{i-1} = s_i - e_i,
// order-isomorphic to the term order on [0, C(n+D, n)): the dictionary of a
// batch is a presence bitmap over that range (fbsp.cu, shard.cu).  `bt` is the
// binomial table bt[x * st + y] = C(x, y), st = n + 1.
#pragma once
#include "common.cuh"

namespace f4b {

static constexpr int MAXV = 32;

template <int KW>
F4B_DEV u32 key_rank(const KeyFmt& f, const u32* bt, int st, const Key<KW>& k) {
  const int n = f.n_vars;
  const int full = (1 << f.lane_bits) - 1;
  const int d = (int)key_lane<KW>(f, k, 0);
  u32 r = d ? bt[(n + d - 1) * st + n] : 0u;
  int s = d;
  for (int L = 1; L < n; ++L) {
    const int i = n - L;
    const int e = full - (int)key_lane<KW>(f, k, L);
    if (s > e) r += bt[(s - e - 1 + i) * st + i];
    s -= e;
  }
  return r;
}

F4B_DEV void unrank_exps(u32 r, int n, int D, const u32* bt, int st, u16* e) {
  // degree: largest d <= D with C(n+d-1, n) <= r  (binary search; C(n-1, n) = 0)
  int lo = 0, hi = D;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bt[(n + mid - 1) * st + n] <= r) lo = mid; else hi = mid - 1;
  }
  const int d = lo;
  if (d) r -= bt[(n + d - 1) * st + n];
  int s = d;
  for (int i = n - 1; i >= 1; --i) {
    // largest m in [0, s] with C(m-1+i, i) <= r  (C(i-1, i) = 0 for m = 0)
    int a = 0, b = s;
    while (a < b) {
      const int mid = (a + b + 1) >> 1;
      if (bt[(mid - 1 + i) * st + i] <= r) a = mid; else b = mid - 1;
    }
    if (a > 0) r -= bt[(a - 1 + i) * st + i];
    e[i] = (u16)(s - a);
    s = a;
  }
  e[0] = (u16)s;
}

// unrank_exps with the exponents in registers (NV >= n, see gl_decode)
template <int NV>
F4B_DEV void gl_unrank(u32 r, int n, int D, const u32* bt, int st, u16 (&e)[NV]) {
  int lo = 0, hi = D;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bt[(n + mid - 1) * st + n] <= r) lo = mid; else hi = mid - 1;
  }
  const int d = lo;
  if (d) r -= bt[(n + d - 1) * st + n];
  int s = d;
#pragma unroll
  for (int i = NV - 1; i >= 1; --i) {
    e[i] = 0;
    if (i < n) {
      int a = 0, b = s;
      while (a < b) {
        const int mid = (a + b + 1) >> 1;
        if (bt[(mid - 1 + i) * st + i] <= r) a = mid; else b = mid - 1;
      }
      if (a > 0) r -= bt[(a - 1 + i) * st + i];
      e[i] = (u16)(s - a);
      s = a;
    }
  }
  e[0] = (u16)s;
}


static inline unsigned long long binom_ull(int a, int b) {
  if (b < 0 || a < b) return 0;
  unsigned long long r = 1;
  for (int i = 1; i <= b; ++i) r = r * (unsigned long long)(a - b + i) / (unsigned long long)i;
  return r;
}

}  // namespace f4b
