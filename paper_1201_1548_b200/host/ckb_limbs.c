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
  for (Py_ssize_t k = 0; k < n; ++k) {
    const uint32_t* c = w + k * lw;
    Py_ssize_t len = lw;
    const uint32_t ext = (c[lw - 1] >> 31) ? 0xffffffffu : 0u;
    /* drop limbs that only repeat the sign, keeping the sign bit in the top one */
    while (len > 1 && c[len - 1] == ext && ((c[len - 2] >> 31) ? 0xffffffffu : 0u) == ext) --len;
    PyObject* v = _PyLong_FromByteArray((const unsigned char*)c, (size_t)(4 * len), 1, 1);
    if (!v) {
      Py_DECREF(out);
      PyBuffer_Release(&view);
      return NULL;
    }
    PyList_SET_ITEM(out, k, v);
  }
  PyBuffer_Release(&view);
  return out;
}

static PyMethodDef methods[] = {
    {"limbs_to_ints", limbs_to_ints, METH_VARARGS, "[N][LW] two's-complement u32 limbs -> list of ints"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "ckb_limbs", NULL, -1, methods};

PyMODINIT_FUNC PyInit_ckb_limbs(void) { return PyModule_Create(&mod); }
