/* Host-side conversion of the engine's output limbs to Python ints.
 *
 * The reference returns list[int] (modpoly.py:348-394); the device writes each
 * coefficient as LW two's-complement little-endian 32-bit limbs.  This builds
 * the list in one C loop, dropping sign-extension limbs first so small
 * coefficients convert in proportion to their size.  (Python-API glue, not
 * part of the compute path.) */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

#if PY_VERSION_HEX >= 0x030C0000 && PY_VERSION_HEX < 0x030E0000 && PyLong_SHIFT == 30
#define CKB_FAST_DIGITS 1
/* Magnitude of a two's-complement limb array repacked straight into CPython's
 * 30-bit digits (_PyLong_FromDigits copies and normalises them): O(limbs),
 * no per-byte loop (_PyLong_FromByteArray costs ~1 us per 5,000-bit
 * coefficient; this ~0.1 us). */
static PyObject* limbs_to_long(const uint32_t* c, Py_ssize_t len, digit* dg, uint32_t* mag) {
  const int neg = (int)(c[len - 1] >> 31);
  const uint32_t* m = c;
  if (neg) { /* magnitude = ~c + 1 */
    uint64_t carry = 1;
    for (Py_ssize_t i = 0; i < len; ++i) {
      const uint64_t v = (uint64_t)(~c[i]) + carry;
      mag[i] = (uint32_t)v;
      carry = v >> 32;
    }
    m = mag;
  }
  Py_ssize_t nd = 0;
  uint64_t acc = 0;
  int bits = 0;
  for (Py_ssize_t i = 0; i < len; ++i) {
    acc |= (uint64_t)m[i] << bits;
    bits += 32;
    while (bits >= PyLong_SHIFT) {
      dg[nd++] = (digit)(acc & PyLong_MASK);
      acc >>= PyLong_SHIFT;
      bits -= PyLong_SHIFT;
    }
  }
  if (bits > 0) dg[nd++] = (digit)(acc & PyLong_MASK);
  while (nd > 0 && dg[nd - 1] == 0) --nd;
  if (nd == 0) return PyLong_FromLong(0);
  return (PyObject*)_PyLong_FromDigits(neg, nd, dg);
}
#endif

static PyObject* limbs_to_ints(PyObject* self, PyObject* args) {
  Py_buffer view;
  Py_ssize_t n, lw;
  if (!PyArg_ParseTuple(args, "y*nn", &view, &n, &lw)) return NULL;
  if (lw < 1 || n < 0 || view.len < (Py_ssize_t)(4 * n * lw)) {
    PyBuffer_Release(&view);
    PyErr_SetString(PyExc_ValueError, "limbs_to_ints: buffer too small");
    return NULL;
  }
  PyObject* out = PyList_New(n);
  if (!out) {
    PyBuffer_Release(&view);
    return NULL;
  }
  const uint32_t* w = (const uint32_t*)view.buf;
#ifdef CKB_FAST_DIGITS
  digit* dg = (digit*)PyMem_Malloc(sizeof(digit) * (size_t)(lw * 32 / PyLong_SHIFT + 2));
  uint32_t* mag = (uint32_t*)PyMem_Malloc(sizeof(uint32_t) * (size_t)lw);
  if (!dg || !mag) {
    PyMem_Free(dg);
    PyMem_Free(mag);
    Py_DECREF(out);
    PyBuffer_Release(&view);
    return PyErr_NoMemory();
  }
#endif
  for (Py_ssize_t k = 0; k < n; ++k) {
    const uint32_t* c = w + k * lw;
    Py_ssize_t len = lw;
    const uint32_t ext = (c[lw - 1] >> 31) ? 0xffffffffu : 0u;
    /* drop limbs that only repeat the sign, keeping the sign bit in the top one */
    while (len > 1 && c[len - 1] == ext && ((c[len - 2] >> 31) ? 0xffffffffu : 0u) == ext) --len;
#ifdef CKB_FAST_DIGITS
    PyObject* v = limbs_to_long(c, len, dg, mag);
#else
    PyObject* v = _PyLong_FromByteArray((const unsigned char*)c, (size_t)(4 * len), 1, 1);
#endif
    if (!v) {
#ifdef CKB_FAST_DIGITS
      PyMem_Free(dg);
      PyMem_Free(mag);
#endif
      Py_DECREF(out);
      PyBuffer_Release(&view);
      return NULL;
    }
    PyList_SET_ITEM(out, k, v);
  }
#ifdef CKB_FAST_DIGITS
  PyMem_Free(dg);
  PyMem_Free(mag);
#endif
  PyBuffer_Release(&view);
  return out;
}

static PyMethodDef methods[] = {
    {"limbs_to_ints", limbs_to_ints, METH_VARARGS, "[N][LW] two's-complement u32 limbs -> list of ints"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "ckb_limbs", NULL, -1, methods};

PyMODINIT_FUNC PyInit_ckb_limbs(void) { return PyModule_Create(&mod); }
