/* Host-side row-list packing for compile_batch (CPython extension).
 *
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
 * Host glue only: nothing here touches the device.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

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

static PyMethodDef methods[] = {
    {"pack_rows", pack_rows, METH_VARARGS, "pack_rows(rows, n, rb_int32, shift_uint16) -> (min_basis, max_basis, lane_ok)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "_rowpack", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__rowpack(void) {
  s_basis_index = PyUnicode_InternFromString("basis_index");
  s_shift = PyUnicode_InternFromString("shift");
  if (!s_basis_index || !s_shift) return NULL;
  return PyModule_Create(&mod);
}
