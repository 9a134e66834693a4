// Shared device definitions for the f4b200 engine (sm_100a).
//
//  * Key<KW>  : a device monomial key — an unsigned integer of 64*KW bits,
//               word 0 most significant.  Order-isomorphic to the reference
//               key (pkg/src/fpgb/monomials.py:137-154) on every monomial of
//               a batch; see paper_2601_06765_b200/monomials.py
//               DeviceKeyFormat for the lane layout.  Shift-multiply is a
//               multiword add of one per-row delta.
//  * Fp       : F_p arithmetic for odd p < 2^31 on u32 residues held in
//               registers: Montgomery with R = 2^32 (reference fp.py:176-185
//               restated for 32-bit lanes).  A scalar is converted into the
//               Montgomery domain once; mont_mul(scalar_m, x_std) then yields
//               a standard-domain product, so all stored data stays standard.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef uint32_t u32;
typedef uint16_t u16;

#define F4B_DEV __device__ __forceinline__
#define F4B_HD __host__ __device__ __forceinline__

// ---------------------------------------------------------------------------
// Multiword keys
// ---------------------------------------------------------------------------
template <int KW>
struct Key {
  u64 w[KW];
};

template <int KW>
F4B_HD bool key_lt(const Key<KW>& a, const Key<KW>& b) {
#pragma unroll
  for (int i = 0; i < KW; ++i) {
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
  }
  return false;
}

template <int KW>
F4B_HD bool key_eq(const Key<KW>& a, const Key<KW>& b) {
  bool e = true;
#pragma unroll
  for (int i = 0; i < KW; ++i) e &= (a.w[i] == b.w[i]);
  return e;
}

// a + b (mod 2^(64 KW)), carries flow from word KW-1 (least significant) up.
template <int KW>
F4B_HD Key<KW> key_add(const Key<KW>& a, const Key<KW>& b) {
  Key<KW> r;
  u64 carry = 0;
#pragma unroll
  for (int i = KW - 1; i >= 0; --i) {
    u64 s = a.w[i] + b.w[i];
    u64 c1 = s < a.w[i];
    u64 s2 = s + carry;
    u64 c2 = s2 < s;
    r.w[i] = s2;
    carry = c1 | c2;
  }
  return r;
}

template <int KW>
F4B_HD Key<KW> key_sub(const Key<KW>& a, const Key<KW>& b) {
  Key<KW> r;
  u64 borrow = 0;
#pragma unroll
  for (int i = KW - 1; i >= 0; --i) {
    u64 d = a.w[i] - b.w[i];
    u64 b1 = a.w[i] < b.w[i];
    u64 d2 = d - borrow;
    u64 b2 = d < borrow;
    r.w[i] = d2;
    borrow = b1 | b2;
  }
  return r;
}

// 8-bit digit at bit offset `bit` counted from the least significant end.
template <int KW>
F4B_HD u32 key_digit(const Key<KW>& k, int bit) {
  // select the word without a dynamic index (a runtime k.w[...] index puts the
  // key array in local memory)
  const int wsel = KW - 1 - (bit >> 6);
  u64 w = k.w[0];
#pragma unroll
  for (int j = 1; j < KW; ++j) w = (j == wsel) ? k.w[j] : w;
  return (u32)((w >> (bit & 63)) & 0xFFu);
}

template <int KW>
F4B_DEV Key<KW> key_load(const u64* __restrict__ base, long long i) {
  Key<KW> k;
  if constexpr (KW == 1) {
    k.w[0] = __ldg(base + i);
  } else if constexpr (KW % 2 == 0) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(base + i * KW);
#pragma unroll
    for (int j = 0; j < KW / 2; ++j) {
      ulonglong2 v = __ldg(p + j);
      k.w[2 * j] = v.x;
      k.w[2 * j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < KW; ++j) k.w[j] = __ldg(base + i * KW + j);
  }
  return k;
}

// Plain (non-__ldg) load for buffers written earlier in the same kernel.
// L2-coherent load (ld.global.cg) for keys written earlier in the SAME
// launch by other CTAs (persistent kernels): never served from a stale L1 line.
template <int KW>
F4B_DEV Key<KW> key_load_cg(const u64* base, long long i) {
  Key<KW> k;
  if constexpr (KW % 2 == 0) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(base + i * KW);
#pragma unroll
    for (int j = 0; j < KW / 2; ++j) {
      const ulonglong2 v = __ldcg(p + j);
      k.w[2 * j] = v.x;
      k.w[2 * j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < KW; ++j) k.w[j] = __ldcg(base + i * KW + j);
  }
  return k;
}

template <int KW>
F4B_DEV Key<KW> key_load_rw(const u64* base, long long i) {
  Key<KW> k;
#pragma unroll
  for (int j = 0; j < KW; ++j) k.w[j] = base[i * KW + j];
  return k;
}

template <int KW>
F4B_DEV void key_store(u64* __restrict__ base, long long i, const Key<KW>& k) {
  if constexpr (KW % 2 == 0) {
    ulonglong2* p = reinterpret_cast<ulonglong2*>(base + i * KW);
#pragma unroll
    for (int j = 0; j < KW / 2; ++j) p[j] = make_ulonglong2(k.w[2 * j], k.w[2 * j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < KW; ++j) base[i * KW + j] = k.w[j];
  }
}

// lower_bound over an ascending key table (global or shared memory).
template <int KW>
F4B_DEV u32 key_lower_bound(const u64* table, u32 n, const Key<KW>& q) {
  u32 lo = 0, hi = n;
  while (lo < hi) {
    u32 mid = (lo + hi) >> 1;
    Key<KW> m = key_load_rw<KW>(table, mid);
    if (key_lt<KW>(m, q)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// Device key format: lane layout (mirrors monomials.DeviceKeyFormat)
// ---------------------------------------------------------------------------
struct KeyFmt {
  int order;      // 0 grevlex, 1 deglex, 2 lex
  int n_vars;
  int lane_bits;  // b
  int n_lanes;    // graded: n_vars (degree + n-1 vars); lex: n_vars
};

// Encode an exponent vector (u16 lanes) into a device key.
template <int KW>
F4B_DEV Key<KW> key_encode(const KeyFmt& f, const u16* e) {
  Key<KW> k;
#pragma unroll
  for (int i = 0; i < KW; ++i) k.w[i] = 0;
  const u32 full = (1u << f.lane_bits) - 1u;
  u32 deg = 0;
  if (f.order != 2) {
    for (int v = 0; v < f.n_vars; ++v) deg += e[v];
  }
  for (int lane = 0; lane < f.n_lanes; ++lane) {
    u32 val;
    if (f.order == 0) val = (lane == 0) ? deg : (full - e[f.n_vars - lane]);
    else if (f.order == 1) val = (lane == 0) ? deg : e[lane - 1];
    else val = e[lane];
    int bit = (f.n_lanes - 1 - lane) * f.lane_bits;  // from the least significant end
    int wi = KW - 1 - (bit >> 6);
    int sh = bit & 63;
    k.w[wi] |= ((u64)val) << sh;
    if (sh + f.lane_bits > 64 && wi > 0) k.w[wi - 1] |= ((u64)val) >> (64 - sh);
  }
  return k;
}

template <int KW>
F4B_DEV u32 key_lane(const KeyFmt& f, const Key<KW>& k, int lane) {
  int bit = (f.n_lanes - 1 - lane) * f.lane_bits;
  int wi = KW - 1 - (bit >> 6);
  int sh = bit & 63;
  // word select without a dynamic index (a runtime k.w[...] index would put
  // the key in local memory)
  u64 lo = k.w[0], hi = 0;
#pragma unroll
  for (int j = 1; j < KW; ++j) {
    if (j == wi) lo = k.w[j];
    if (j == wi - 1) hi = k.w[j];
  }
  u64 v = lo >> sh;
  if (KW > 1 && sh + f.lane_bits > 64 && wi > 0) v |= hi << (64 - sh);
  return (u32)(v & ((1ull << f.lane_bits) - 1ull));
}

// OR a lane value into a key (lane counted from the most significant end).
template <int KW>
F4B_DEV void key_or_lane(const KeyFmt& f, Key<KW>& k, int lane, u32 val) {
  const int bit = (f.n_lanes - 1 - lane) * f.lane_bits;
  const int wi = KW - 1 - (bit >> 6);
  const int sh = bit & 63;
#pragma unroll
  for (int j = 0; j < KW; ++j) {
    if (j == wi) k.w[j] |= ((u64)val) << sh;
    if (KW > 1 && j == wi - 1 && sh + f.lane_bits > 64) k.w[j] |= ((u64)val) >> (64 - sh);
  }
}

// ---- grevlex keys with a compile-time bound NV >= n_vars on the number of
// variables: exponent vectors live in registers (every index is a
// compile-time constant after unrolling), no local-memory frame.
// grevlex lanes: lane 0 = degree, lane L (1 <= L < n) = full - e_{n-L}.
template <int KW, int NV>
F4B_DEV void gl_decode(const KeyFmt& f, const Key<KW>& k, u16 (&e)[NV]) {
  const u32 full = (1u << f.lane_bits) - 1u;
  const int n = f.n_vars;
  u32 rest = 0;
#pragma unroll
  for (int v = 1; v < NV; ++v) {
    e[v] = 0;
    if (v < n) {
      const u32 x = full - key_lane<KW>(f, k, n - v);
      e[v] = (u16)x;
      rest += x;
    }
  }
  e[0] = (u16)(key_lane<KW>(f, k, 0) - rest);
}

template <int KW, int NV>
F4B_DEV Key<KW> gl_encode(const KeyFmt& f, const u16 (&e)[NV]) {
  Key<KW> k;
#pragma unroll
  for (int j = 0; j < KW; ++j) k.w[j] = 0;
  const u32 full = (1u << f.lane_bits) - 1u;
  const int n = f.n_vars;
  u32 deg = 0;
#pragma unroll
  for (int v = 0; v < NV; ++v)
    if (v < n) deg += e[v];
  key_or_lane<KW>(f, k, 0, deg);
#pragma unroll
  for (int v = 1; v < NV; ++v)
    if (v < n) key_or_lane<KW>(f, k, n - v, full - e[v]);
  return k;
}

// Decode a device key into exponents.
template <int KW>
F4B_DEV void key_decode(const KeyFmt& f, const Key<KW>& k, u16* e) {
  const u32 full = (1u << f.lane_bits) - 1u;
  if (f.order == 2) {
    for (int v = 0; v < f.n_vars; ++v) e[v] = (u16)key_lane<KW>(f, k, v);
    return;
  }
  u32 deg = key_lane<KW>(f, k, 0);
  u32 rest = 0;
  for (int lane = 1; lane < f.n_lanes; ++lane) {
    u32 l = key_lane<KW>(f, k, lane);
    u32 ex = (f.order == 0) ? (full - l) : l;
    int v = (f.order == 0) ? (f.n_vars - lane) : (lane - 1);
    e[v] = (u16)ex;
    rest += ex;
  }
  int implied = (f.order == 0) ? 0 : (f.n_vars - 1);
  e[implied] = (u16)(deg - rest);
}

// ---------------------------------------------------------------------------
// F_p arithmetic (u32 residues, Montgomery R = 2^32)
// ---------------------------------------------------------------------------
struct Fp {
  u32 p;
  u32 pprime;  // p * pprime == -1 (mod 2^32)
  u32 r2;      // 2^64 mod p

  F4B_HD u32 mont_mul(u32 a, u32 b) const {
    u64 t = (u64)a * b;
    u32 m = (u32)t * pprime;
    u64 u = (t + (u64)m * p) >> 32;
    return (u32)(u >= p ? u - p : u);
  }
  F4B_HD u32 to_mont(u32 a) const { return mont_mul(a, r2); }
  // standard-domain product
  F4B_HD u32 mul(u32 a, u32 b) const { return mont_mul(to_mont(a), b); }
  F4B_HD u32 add(u32 a, u32 b) const {
    u32 s = a + b;
    return s >= p ? s - p : s;
  }
  F4B_HD u32 sub(u32 a, u32 b) const { return a >= b ? a - b : a + p - b; }
  F4B_HD u32 neg(u32 a) const { return a ? p - a : 0; }
  // a^(p-2) (a != 0), standard domain in and out
  F4B_HD u32 inv(u32 a) const {
    u32 base = to_mont(a);
    u32 acc = to_mont(1);
    u32 e = p - 2;
    while (e) {
      if (e & 1) acc = mont_mul(acc, base);
      base = mont_mul(base, base);
      e >>= 1;
    }
    return mont_mul(acc, 1);  // leave the Montgomery domain
  }
};

// ---------------------------------------------------------------------------
// Error flags written by kernels (bit set -> C-ABI status code)
// ---------------------------------------------------------------------------
enum DevErr : u32 {
  DEVERR_MISSING_KEY = 1u,
  DEVERR_LANE_OVERFLOW = 2u,
  DEVERR_ZERO_REDUCER = 4u,
  DEVERR_CAPACITY = 8u,
};

F4B_DEV unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
