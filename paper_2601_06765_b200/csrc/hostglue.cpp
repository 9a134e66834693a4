/* Host glue of the F4 driver (CPython extension, C++; no device code):
 *
 *   pack_rows      compile_batch's Row list -> flat arrays (below)
 *   gm_new_pairs   Gebauer-Moeller criteria on the pairs (i, t) of a new
 *   gm_prune       basis element t, and on the queued pairs (update_pairs)
 *
 * Row packing.
 * The reference's compile_batch (pkg/src/fpgb/symbolic.py:293-388) takes its
 * rows as a list of Row objects (shift tuple, basis index, role, provenance).
 * The device path needs them as two flat arrays: the basis index of every row
 * (int32) and its shift exponents (u16 lanes, n per row).  Walking the list
 * in Python (attrgetter + itertools.chain + numpy.fromiter) costs ~60 ns per
 * exponent; this walks it in C over the object pointers.
 *
 *   pack_rows(rows, n, rb, sh) -> (min_basis, max_basis, lane_ok)
 *
 * rows: a sequence of objects with .basis_index (int) and .shift (sequence
 * of n ints); rb: writable buffer of len(rows) int32; sh: writable buffer of
 * len(rows) * n uint16.  lane_ok is False when a shift exponent is negative
 * or above 0xFFFF (the caller raises LaneOverflowError, monomials.py lanes);
 * the caller range-checks the basis indices (IndexError, as before).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

#include <algorithm>
#include <numeric>
#include <vector>

static PyObject* s_basis_index;
static PyObject* s_shift;

static PyObject* pack_rows(PyObject* self, PyObject* args) {
  (void)self;
  PyObject* seq;
  Py_ssize_t n;
  Py_buffer rb, sh;
  if (!PyArg_ParseTuple(args, "Onw*w*", &seq, &n, &rb, &sh)) return NULL;
  PyObject* fast = PySequence_Fast(seq, "rows must be a sequence");
  if (!fast) {
    PyBuffer_Release(&rb);
    PyBuffer_Release(&sh);
    return NULL;
  }
  const Py_ssize_t R = PySequence_Fast_GET_SIZE(fast);
  PyObject* ret = NULL;
  if (n < 1 || rb.len < R * (Py_ssize_t)sizeof(int32_t) || sh.len < R * n * (Py_ssize_t)sizeof(uint16_t)) {
    PyErr_SetString(PyExc_ValueError, "pack_rows: output buffers too small");
    goto done;
  }
  {
    int32_t* orb = (int32_t*)rb.buf;
    uint16_t* osh = (uint16_t*)sh.buf;
    PyObject** items = PySequence_Fast_ITEMS(fast);
    long long bmin = 0, bmax = -1;
    int lane_ok = 1;
    for (Py_ssize_t i = 0; i < R; ++i) {
      PyObject* row = items[i];
      PyObject* b = PyObject_GetAttr(row, s_basis_index);
      if (!b) goto done;
      const long long bi = PyLong_AsLongLong(b);
      Py_DECREF(b);
      if (bi == -1 && PyErr_Occurred()) goto done;
      if (i == 0 || bi < bmin) bmin = bi;
      if (i == 0 || bi > bmax) bmax = bi;
      orb[i] = (bi < INT32_MIN || bi > INT32_MAX) ? -1 : (int32_t)bi;  // out of range: caught by the caller's bounds
      PyObject* t = PyObject_GetAttr(row, s_shift);
      if (!t) goto done;
      PyObject* tf = PyTuple_CheckExact(t) ? (Py_INCREF(t), t) : PySequence_Fast(t, "shift must be a sequence");
      Py_DECREF(t);
      if (!tf) goto done;
      if (PySequence_Fast_GET_SIZE(tf) != n) {
        Py_DECREF(tf);
        PyErr_SetString(PyExc_ValueError, "shift length differs from the ring's variable count");
        goto done;
      }
      PyObject** ev = PySequence_Fast_ITEMS(tf);
      uint16_t* o = osh + i * n;
      for (Py_ssize_t k = 0; k < n; ++k) {
        const long long e = PyLong_AsLongLong(ev[k]);
        if (e == -1 && PyErr_Occurred()) {
          Py_DECREF(tf);
          goto done;
        }
        if (e < 0 || e > 0xFFFF) lane_ok = 0;
        o[k] = (uint16_t)e;
      }
      Py_DECREF(tf);
    }
    ret = Py_BuildValue("LLO", bmin, bmax, lane_ok ? Py_True : Py_False);
  }
done:
  Py_DECREF(fast);
  PyBuffer_Release(&rb);
  PyBuffer_Release(&sh);
  return ret;
}

/* ---------------------------------------------------------------------------
 * Gebauer-Moeller update (reference groebner.py:154-201; the NumPy statement
 * is in tests/test_host.py).  The pair logic reads leading monomials only
 * (SURVEY 8f.2).
 *
 * New pairs (i, t) of basis element t with leading exponents lm, partners
 * i < t with leading exponents L_i, lcm_i = max(L_i, lm): partner i survives
 * when lcm_i is minimal among the distinct lcms (divisible by no other one),
 * i is the lowest partner index of its lcm, and gcd(L_i, lm) != 1 (product
 * criterion on the representative).  Surviving partners ascending.
 * ------------------------------------------------------------------------- */
static void new_pairs_impl(const int64_t* L, Py_ssize_t t, Py_ssize_t n, const int64_t* lm, std::vector<int64_t>& surv) {
  surv.clear();
  std::vector<int64_t> lcm((size_t)t * n);
  struct Ent {
    int64_t deg;
    uint64_t pk;  // the row packed 8 bits per variable (when it fits) for a flat compare
    int32_t i;
  };
  std::vector<Ent> ent((size_t)t);
  bool packable = n <= 8;
  for (Py_ssize_t i = 0; i < t; ++i) {
    int64_t d = 0;
    uint64_t pk = 0;
    for (Py_ssize_t v = 0; v < n; ++v) {
      const int64_t x = std::max(L[i * n + v], lm[v]);
      lcm[(size_t)i * n + v] = x;
      d += x;
      packable = packable && x >= 0 && x < 256;
      pk = (pk << 8) | (uint64_t)(x & 0xFF);
    }
    ent[i] = {d, pk, (int32_t)i};
  }
  auto row = [&](int32_t i) { return &lcm[(size_t)i * n]; };
  if (packable) {
    std::sort(ent.begin(), ent.end(), [](const Ent& a, const Ent& b) {
      return a.deg != b.deg ? a.deg < b.deg : (a.pk != b.pk ? a.pk < b.pk : a.i < b.i);
    });
  } else {
    std::sort(ent.begin(), ent.end(), [&](const Ent& a, const Ent& b) {
      if (a.deg != b.deg) return a.deg < b.deg;
      const int64_t *x = row(a.i), *y = row(b.i);
      for (Py_ssize_t v = 0; v < n; ++v)
        if (x[v] != y[v]) return x[v] < y[v];
      return a.i < b.i;
    });
  }
  std::vector<int32_t> kept;  // one representative per minimal lcm, ascending degree
  for (Py_ssize_t s0 = 0; s0 < t;) {
    const int32_t rep = ent[s0].i;  // lowest index of this lcm
    const int64_t* x = row(rep);
    Py_ssize_t e = s0 + 1;
    while (e < t && ent[e].deg == ent[s0].deg && std::equal(x, x + n, row(ent[e].i))) ++e;
    bool dom = false;
    for (int32_t k : kept) {  // a minimal lcm of smaller degree dividing this one
      const int64_t* y = row(k);
      Py_ssize_t v = 0;
      while (v < n && y[v] <= x[v]) ++v;
      if (v == n) {
        dom = true;
        break;
      }
    }
    if (!dom) {
      kept.push_back(rep);
      bool coprime = true;
      for (Py_ssize_t v = 0; v < n && coprime; ++v) coprime = std::min(L[(size_t)rep * n + v], lm[v]) == 0;
      if (!coprime) surv.push_back(rep);
    }
    s0 = e;
  }
  std::sort(surv.begin(), surv.end());
}

/* Chain criterion on the queued pairs: pair q = (i, j) with lcm l is dropped
 * when lm | l, max(L_i, lm) != l and max(L_j, lm) != l.  keep[q] = 1 stays.
 * Returns false on a pair index outside [0, nL). */
static bool prune_impl(const int64_t* pl, const int64_t* pi, const int64_t* pj, Py_ssize_t P, const int64_t* L,
                       Py_ssize_t nL, Py_ssize_t n, const int64_t* lm, uint8_t* keep) {
  for (Py_ssize_t q = 0; q < P; ++q) {
    const int64_t* l = pl + q * n;
    bool hit = true;
    for (Py_ssize_t v = 0; v < n && hit; ++v) hit = l[v] >= lm[v];
    if (hit) {
      if (pi[q] < 0 || pi[q] >= nL || pj[q] < 0 || pj[q] >= nL) return false;
      const int64_t* a = L + pi[q] * n;
      const int64_t* b = L + pj[q] * n;
      bool da = false, db = false;
      for (Py_ssize_t v = 0; v < n; ++v) {
        da |= std::max(a[v], lm[v]) != l[v];
        db |= std::max(b[v], lm[v]) != l[v];
      }
      hit = da && db;
    }
    keep[q] = hit ? 0 : 1;
  }
  return true;
}

// gm_new_pairs(L, t, n, lm, surv_out) -> count
static PyObject* gm_new_pairs(PyObject* self, PyObject* args) {
  (void)self;
  Py_buffer bL, blm, bs;
  Py_ssize_t t, n;
  if (!PyArg_ParseTuple(args, "y*nny*w*", &bL, &t, &n, &blm, &bs)) return NULL;
  PyObject* ret = NULL;
  if (t < 0 || n < 1 || bL.len < t * n * 8 || blm.len < n * 8 || bs.len < t * 8) {
    PyErr_SetString(PyExc_ValueError, "gm_new_pairs: buffer sizes");
  } else {
    std::vector<int64_t> surv;
    new_pairs_impl((const int64_t*)bL.buf, t, n, (const int64_t*)blm.buf, surv);
    std::copy(surv.begin(), surv.end(), (int64_t*)bs.buf);
    ret = PyLong_FromSsize_t((Py_ssize_t)surv.size());
  }
  PyBuffer_Release(&bL);
  PyBuffer_Release(&blm);
  PyBuffer_Release(&bs);
  return ret;
}

// gm_prune(plcm, pi, pj, P, L, n, lm, keep_out) -> kept count
static PyObject* gm_prune(PyObject* self, PyObject* args) {
  (void)self;
  Py_buffer bl, bi, bj, bL, blm, bk;
  Py_ssize_t P, n;
  if (!PyArg_ParseTuple(args, "y*y*y*ny*ny*w*", &bl, &bi, &bj, &P, &bL, &n, &blm, &bk)) return NULL;
  PyObject* ret = NULL;
  if (P < 0 || n < 1 || bl.len < P * n * 8 || bi.len < P * 8 || bj.len < P * 8 || blm.len < n * 8 || bk.len < P) {
    PyErr_SetString(PyExc_ValueError, "gm_prune: buffer sizes");
  } else {
    uint8_t* keep = (uint8_t*)bk.buf;
    if (!prune_impl((const int64_t*)bl.buf, (const int64_t*)bi.buf, (const int64_t*)bj.buf, P,
                    (const int64_t*)bL.buf, bL.len / (n * 8), n, (const int64_t*)blm.buf, keep)) {
      PyErr_SetString(PyExc_IndexError, "gm_prune: pair index outside the basis");
    } else {
      Py_ssize_t kept = 0;
      for (Py_ssize_t q = 0; q < P; ++q) kept += keep[q];
      ret = PyLong_FromSsize_t(kept);
    }
  }
  PyBuffer_Release(&bl);
  PyBuffer_Release(&bi);
  PyBuffer_Release(&bj);
  PyBuffer_Release(&bL);
  PyBuffer_Release(&blm);
  PyBuffer_Release(&bk);
  return ret;
}

/* gm_update(L, t, n, lm, graded, grevlex, W,
 *           pi, pj, plcm, pdeg, pkey, P,
 *           o_pi, o_pj, o_plcm, o_pdeg, o_pkey) -> count, or -1 on lane overflow
 * The whole update_pairs queue step: the queued pairs (sorted by
 * (degree, key(lcm), i, j), reference Pair.sort_tuple, groebner.py:110-116)
 * minus the chain-criterion hits, merged with the surviving new pairs
 * (i, t) in the same order.  key(lcm) is the reference monomial key
 * (monomials.py mon_key_pack: [32-bit degree if graded] then 16-bit lanes,
 * grevlex lanes 0xFFFF - e in reversed variable order, most significant
 * word first).  Outputs hold P + t entries. */
static PyObject* gm_update(PyObject* self, PyObject* args) {
  (void)self;
  Py_buffer bL, blm, bi, bj, bl, bd, bk, oi, oj, ol, od, ok;
  Py_ssize_t t, n, W, P;
  int graded, grevlex;
  if (!PyArg_ParseTuple(args, "y*nny*iiny*y*y*y*y*nw*w*w*w*w*", &bL, &t, &n, &blm, &graded, &grevlex, &W, &bi, &bj,
                        &bl, &bd, &bk, &P, &oi, &oj, &ol, &od, &ok))
    return NULL;
  Py_buffer* all[] = {&bL, &blm, &bi, &bj, &bl, &bd, &bk, &oi, &oj, &ol, &od, &ok};
  PyObject* ret = NULL;
  const Py_ssize_t cap = P + t;
  if (t < 0 || P < 0 || n < 1 || W < 1 || bL.len < t * n * 8 || blm.len < n * 8 || bi.len < P * 8 ||
      bj.len < P * 8 || bl.len < P * n * 8 || bd.len < P * 8 || bk.len < P * W * 8 || oi.len < cap * 8 ||
      oj.len < cap * 8 || ol.len < cap * n * 8 || od.len < cap * 8 || ok.len < cap * W * 8 ||
      (graded ? 32 : 0) + 16 * n > 64 * W) {
    PyErr_SetString(PyExc_ValueError, "gm_update: buffer sizes");
  } else {
    const int64_t* L = (const int64_t*)bL.buf;
    const int64_t* lm = (const int64_t*)blm.buf;
    const int64_t* pi = (const int64_t*)bi.buf;
    const int64_t* pj = (const int64_t*)bj.buf;
    const int64_t* pl = (const int64_t*)bl.buf;
    const int64_t* pd = (const int64_t*)bd.buf;
    const uint64_t* pk = (const uint64_t*)bk.buf;
    int64_t* Oi = (int64_t*)oi.buf;
    int64_t* Oj = (int64_t*)oj.buf;
    int64_t* Ol = (int64_t*)ol.buf;
    int64_t* Od = (int64_t*)od.buf;
    uint64_t* Ok = (uint64_t*)ok.buf;
    std::vector<int64_t> surv;
    new_pairs_impl(L, t, n, lm, surv);
    std::vector<uint8_t> keep((size_t)P);
    if (!prune_impl(pl, pi, pj, P, L, t, n, lm, keep.data())) {
      PyErr_SetString(PyExc_IndexError, "gm_update: pair index outside the basis");
    } else {
      // the new pairs' lcm, degree and key, sorted by (degree, key, i)
      const size_t ns = surv.size();
      std::vector<int64_t> nl(ns * n), nd(ns);
      std::vector<uint64_t> nk(ns * W, 0);
      bool overflow = false;
      for (size_t q = 0; q < ns; ++q) {
        int64_t d = 0;
        for (Py_ssize_t v = 0; v < n; ++v) {
          const int64_t x = std::max(L[surv[q] * n + v], lm[v]);
          nl[q * n + v] = x;
          d += x;
          overflow |= x < 0 || x > 0xFFFF;
        }
        nd[q] = d;
        overflow |= graded && (d >> 32) != 0;
        uint64_t* key = &nk[q * W];
        const int head = graded ? 32 : 0;
        if (graded) key[0] |= (uint64_t)d << 32;
        for (Py_ssize_t i = 0; i < n; ++i) {
          const uint64_t lane = grevlex ? (uint64_t)(0xFFFF - nl[q * n + (n - 1 - i)]) : (uint64_t)nl[q * n + i];
          const int off = head + 16 * (int)i;
          key[off / 64] |= (lane & 0xFFFF) << (64 - off % 64 - 16);
        }
      }
      if (overflow) {
        ret = PyLong_FromLong(-1);
      } else {
        auto key_less = [&](int64_t da, const uint64_t* ka, int64_t ia, int64_t ja, int64_t db, const uint64_t* kb,
                            int64_t ib, int64_t jb) {
          if (da != db) return da < db;
          for (Py_ssize_t w = 0; w < W; ++w)
            if (ka[w] != kb[w]) return ka[w] < kb[w];
          if (ia != ib) return ia < ib;
          return ja < jb;
        };
        std::vector<size_t> ord(ns);
        std::iota(ord.begin(), ord.end(), 0);
        std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
          return key_less(nd[a], &nk[a * W], surv[a], t, nd[b], &nk[b * W], surv[b], t);
        });
        // merge (old kept pairs are already in order; ties keep the old pair first, as the stable sort did)
        Py_ssize_t m = 0, q = 0;
        size_t r = 0;
        auto emit_old = [&](Py_ssize_t x) {
          Oi[m] = pi[x];
          Oj[m] = pj[x];
          std::copy(pl + x * n, pl + (x + 1) * n, Ol + m * n);
          Od[m] = pd[x];
          std::copy(pk + x * W, pk + (x + 1) * W, Ok + m * W);
          ++m;
        };
        auto emit_new = [&](size_t y) {
          Oi[m] = surv[y];
          Oj[m] = t;
          std::copy(&nl[y * n], &nl[(y + 1) * n], Ol + m * n);
          Od[m] = nd[y];
          std::copy(&nk[y * W], &nk[(y + 1) * W], Ok + m * W);
          ++m;
        };
        while (true) {
          while (q < P && !keep[q]) ++q;
          if (q >= P || r >= ns) break;
          const size_t y = ord[r];
          if (key_less(nd[y], &nk[y * W], surv[y], t, pd[q], pk + q * W, pi[q], pj[q])) {
            emit_new(y);
            ++r;
          } else {
            emit_old(q);
            ++q;
          }
        }
        for (; q < P; ++q)
          if (keep[q]) emit_old(q);
        for (; r < ns; ++r) emit_new(ord[r]);
        ret = PyLong_FromSsize_t(m);
      }
    }
  }
  for (Py_buffer* b : all) PyBuffer_Release(b);
  return ret;
}

/* pack_keys(exps, K, n, graded, grevlex, W, out) -> 0 | 1 (lane overflow) |
 * 2 (degree overflow): the reference keys of K exponent rows (monomials.py
 * key_pack_vec / mon_key_pack), out uint64 [K][W]. */
static PyObject* pack_keys(PyObject* self, PyObject* args) {
  (void)self;
  Py_buffer be, bo;
  Py_ssize_t K, n, W;
  int graded, grevlex;
  if (!PyArg_ParseTuple(args, "y*nniinw*", &be, &K, &n, &graded, &grevlex, &W, &bo)) return NULL;
  PyObject* ret = NULL;
  if (K < 0 || n < 1 || W < 1 || be.len < K * n * 8 || bo.len < K * W * 8 || (graded ? 32 : 0) + 16 * n > 64 * W) {
    PyErr_SetString(PyExc_ValueError, "pack_keys: buffer sizes");
  } else {
    const int64_t* e = (const int64_t*)be.buf;
    uint64_t* out = (uint64_t*)bo.buf;
    const int head = graded ? 32 : 0;
    long code = 0;
    Py_BEGIN_ALLOW_THREADS
    for (Py_ssize_t t = 0; t < K && !code; ++t) {
      const int64_t* x = e + t * n;
      uint64_t* k = out + t * W;
      for (Py_ssize_t w = 0; w < W; ++w) k[w] = 0;
      uint64_t deg = 0;
      for (Py_ssize_t v = 0; v < n; ++v) {
        if (x[v] < 0 || x[v] > 0xFFFF) {
          code = 1;
          break;
        }
        deg += (uint64_t)x[v];
      }
      if (code) break;
      if (graded) {
        if (deg >> 32) {
          code = 2;
          break;
        }
        k[0] |= deg << 32;
      }
      for (Py_ssize_t i = 0; i < n; ++i) {
        const uint64_t lane = grevlex ? 0xFFFFu - (uint64_t)x[n - 1 - i] : (uint64_t)x[i];
        const int off = head + 16 * (int)i;
        k[off >> 6] |= lane << (48 - (off & 63));
      }
    }
    Py_END_ALLOW_THREADS
    ret = PyLong_FromLong(code);
  }
  PyBuffer_Release(&be);
  PyBuffer_Release(&bo);
  return ret;
}

static PyMethodDef methods[] = {
    {"pack_keys", pack_keys, METH_VARARGS, "pack_keys(exps, K, n, graded, grevlex, W, out) -> 0 | 1 | 2"},
    {"pack_rows", pack_rows, METH_VARARGS, "pack_rows(rows, n, rb_int32, shift_uint16) -> (min_basis, max_basis, lane_ok)"},
    {"gm_new_pairs", gm_new_pairs, METH_VARARGS, "gm_new_pairs(L, t, n, lm, surv_out) -> count"},
    {"gm_prune", gm_prune, METH_VARARGS, "gm_prune(plcm, pi, pj, P, L, n, lm, keep_out) -> kept"},
    {"gm_update", gm_update, METH_VARARGS,
     "gm_update(L, t, n, lm, graded, grevlex, W, pi, pj, plcm, pdeg, pkey, P, o_pi, o_pj, o_plcm, o_pdeg, o_pkey) -> count"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_hostglue", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__hostglue(void) {
  s_basis_index = PyUnicode_InternFromString("basis_index");
  s_shift = PyUnicode_InternFromString("shift");
  if (!s_basis_index || !s_shift) return NULL;
  return PyModule_Create(&mod);
}
