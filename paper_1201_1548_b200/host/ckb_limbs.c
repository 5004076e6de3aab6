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
/* the magnitude's digits into dg (room for len * 32 / 30 + 2), returns the
 * normalised digit count; *neg = sign (no Python API: runs without the GIL) */
static Py_ssize_t limbs_to_digits(const uint32_t* c, Py_ssize_t len, digit* dg, int* negp) {
  const int neg = (int)(c[len - 1] >> 31);
  /* magnitude = (c ^ flip) + carry0, negated on the fly for a negative value */
  const uint32_t flip = neg ? 0xffffffffu : 0u;
  uint64_t carry = neg ? 1u : 0u;
  Py_ssize_t nd = 0;
  Py_ssize_t i = 0;
  /* 15 limbs = 480 bits = 16 digits: a fixed shift pattern the compiler unrolls */
  for (; i + 15 <= len; i += 15) {
    uint32_t s[15];
#pragma GCC unroll 15
    for (int k = 0; k < 15; ++k) {
      const uint64_t v = (uint64_t)(c[i + k] ^ flip) + carry;
      s[k] = (uint32_t)v;
      carry = v >> 32;
    }
    digit* d = dg + nd;
#pragma GCC unroll 16
    for (int t = 0; t < 16; ++t) {
      const int bit = 30 * t, w = bit >> 5, o = bit & 31;
      uint64_t v = (uint64_t)s[w] >> o;
      if (o > 2 && w + 1 < 15) v |= (uint64_t)s[w + 1] << (32 - o);
      d[t] = (digit)(v & PyLong_MASK);
    }
    nd += 16;
  }
  uint64_t acc = 0;
  int bits = 0;
  for (; i < len; ++i) {
    const uint64_t v = (uint64_t)(c[i] ^ flip) + carry;
    carry = v >> 32;
    acc |= (uint64_t)(uint32_t)v << bits;
    bits += 32;
    while (bits >= PyLong_SHIFT) {
      dg[nd++] = (digit)(acc & PyLong_MASK);
      acc >>= PyLong_SHIFT;
      bits -= PyLong_SHIFT;
    }
  }
  if (bits > 0) dg[nd++] = (digit)(acc & PyLong_MASK);
  while (nd > 0 && dg[nd - 1] == 0) --nd;
  *negp = neg;
  return nd;
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
  /* pass 1: one int object per coefficient, allocated for the largest digit
   * count its limbs allow; pass 2 (GIL released): the digits written straight
   * into the objects (no staging buffer, no copy), then normalised.  The
   * objects are not visible to Python until the list is returned.  (Worker
   * threads for pass 2 measured erratic on CPU-quota'd hosts: not used.) */
  Py_ssize_t* lens = (Py_ssize_t*)PyMem_Malloc(sizeof(Py_ssize_t) * (size_t)(n ? n : 1));
  if (!lens) {
    Py_DECREF(out);
    PyBuffer_Release(&view);
    return PyErr_NoMemory();
  }
  for (Py_ssize_t k = 0; k < n; ++k) {
    const uint32_t* c = w + k * lw;
    Py_ssize_t len = lw;
    const uint32_t ext = (c[lw - 1] >> 31) ? 0xffffffffu : 0u;
    while (len > 1 && c[len - 1] == ext && ((c[len - 2] >> 31) ? 0xffffffffu : 0u) == ext) --len;
    lens[k] = len;
    PyObject* v;
    if (len == 1 && c[0] == 0u) {
      v = PyLong_FromLong(0);
      lens[k] = 0;  /* nothing to fill */
    } else {
      v = (PyObject*)_PyLong_New(len * 32 / PyLong_SHIFT + 2);
    }
    if (!v) {
      PyMem_Free(lens);
      Py_DECREF(out);
      PyBuffer_Release(&view);
      return NULL;
    }
    PyList_SET_ITEM(out, k, v);
  }
  PyObject** items = ((PyListObject*)out)->ob_item;
  Py_BEGIN_ALLOW_THREADS
  for (Py_ssize_t k = 0; k < n; ++k) {
    if (!lens[k]) continue;
    PyLongObject* v = (PyLongObject*)items[k];
    int neg = 0;
    const Py_ssize_t nd = limbs_to_digits(w + k * lw, lens[k], v->long_value.ob_digit, &neg);
    /* lv_tag = digit count << 3 | sign (0: positive, 1: zero, 2: negative) */
    v->long_value.lv_tag = nd ? ((uintptr_t)nd << 3) | (neg ? 2u : 0u) : 1u;
    if (!nd) v->long_value.ob_digit[0] = 0;
  }
  Py_END_ALLOW_THREADS
  PyMem_Free(lens);
#else
  for (Py_ssize_t k = 0; k < n; ++k) {
    const uint32_t* c = w + k * lw;
    Py_ssize_t len = lw;
    const uint32_t ext = (c[lw - 1] >> 31) ? 0xffffffffu : 0u;
    while (len > 1 && c[len - 1] == ext && ((c[len - 2] >> 31) ? 0xffffffffu : 0u) == ext) --len;
    PyObject* v = _PyLong_FromByteArray((const unsigned char*)c, (size_t)(4 * len), 1, 1);
    if (!v) {
      Py_DECREF(out);
      PyBuffer_Release(&view);
      return NULL;
    }
    PyList_SET_ITEM(out, k, v);
  }
#endif
  PyBuffer_Release(&view);
  return out;
}

/* ------------------------------------------------------------------------
 * terms_grid(terms_f, terms_g, swap): the input side of the same glue.
 *
 * Reads two {(i, j): c} term dicts (the reference's BivPoly.terms,
 * bivpoly.py:18-25; i = power of x, j = power of y; swap exchanges them for
 * res_x) in one C pass each and returns what planner.pack_grid and
 * planner.plan_resultant would derive from coeffs_wrt_y (bivpoly.py:71-80):
 *   (limbs: bytes, L, m, n, dfx, dgx, tdf, tdg, degs: bytes (int16),
 *    norm1: list[float] | None, lcf: list[int], lcg: list[int])
 * with the limb grid in pack_grid's layout (f's y-rows padded to dfx + 1
 * coefficients, then g's to dgx + 1; L two's-complement u32 limbs each) and
 * norm1 the per-row 1-norms as doubles (None if one overflows a double).
 * Returns None when the input is not in that plain form (non-dict, non-int
 * keys or coefficients, negative exponents): the caller takes the Python path.
 * ------------------------------------------------------------------------ */
typedef struct {
  Py_ssize_t rows; /* deg_y + 1 */
  Py_ssize_t dx;   /* max x-degree over rows */
  long td;         /* total degree */
  int16_t* deg;    /* [rows] trimmed x-degree per row, -1 for an empty row */
  double* norm;    /* [rows] */
  int norm_ok;
} GridSide;

static int key_ij(PyObject* key, int swap, long* i, long* j) {
  if (!PyTuple_CheckExact(key) || PyTuple_GET_SIZE(key) != 2) return 0;
  PyObject* a = PyTuple_GET_ITEM(key, 0);
  PyObject* b = PyTuple_GET_ITEM(key, 1);
  if (!PyLong_CheckExact(a) || !PyLong_CheckExact(b)) return 0;
  const long x = PyLong_AsLong(a), y = PyLong_AsLong(b);
  if ((x == -1 || y == -1) && PyErr_Occurred()) {
    PyErr_Clear();
    return 0;
  }
  if (x < 0 || y < 0 || x > 1000000 || y > 1000000) return 0;
  *i = swap ? y : x;
  *j = swap ? x : y;
  return 1;
}

/* pass 1: shape, degrees, 1-norms and the widest coefficient; 0 = not plain */
static int scan_side(PyObject* terms, int swap, GridSide* s, size_t* maxbits) {
  Py_ssize_t pos = 0;
  PyObject *k, *v;
  long i, j, maxj = -1, maxi = -1;
  s->td = -1;
  while (PyDict_Next(terms, &pos, &k, &v)) {
    if (!PyLong_CheckExact(v) || !key_ij(k, swap, &i, &j)) return 0;
    if (_PyLong_Sign(v) == 0) continue;
    if (j > maxj) maxj = j;
    if (i > maxi) maxi = i;
    if (i + j > s->td) s->td = i + j;
  }
  s->rows = maxj + 1;
  s->dx = maxi < 0 ? 0 : maxi;
  s->deg = (int16_t*)PyMem_Malloc(sizeof(int16_t) * (size_t)(s->rows > 0 ? s->rows : 1));
  s->norm = (double*)PyMem_Calloc((size_t)(s->rows > 0 ? s->rows : 1), sizeof(double));
  if (!s->deg || !s->norm) return -1;
  for (Py_ssize_t r = 0; r < s->rows; ++r) s->deg[r] = -1;
  s->norm_ok = 1;
  pos = 0;
  while (PyDict_Next(terms, &pos, &k, &v)) {
    key_ij(k, swap, &i, &j);
    if (_PyLong_Sign(v) == 0) continue;
    if (i > s->deg[j]) s->deg[j] = (int16_t)i;
    const size_t nb = _PyLong_NumBits(v);
    if (nb > *maxbits) *maxbits = nb;
    if (s->norm_ok) {
      const double d = PyLong_AsDouble(v);
      if (d == -1.0 && PyErr_Occurred()) {
        PyErr_Clear();
        s->norm_ok = 0;
      } else {
        s->norm[j] += d < 0 ? -d : d;
      }
    }
  }
  return 1;
}

/* pass 2: every nonzero coefficient into its grid slot */
static int write_side(PyObject* terms, int swap, Py_ssize_t dx, Py_ssize_t L, unsigned char* base) {
  Py_ssize_t pos = 0;
  PyObject *k, *v;
  long i, j;
  while (PyDict_Next(terms, &pos, &k, &v)) {
    key_ij(k, swap, &i, &j);
    if (_PyLong_Sign(v) == 0) continue;
    unsigned char* dst = base + ((size_t)j * (size_t)(dx + 1) + (size_t)i) * (size_t)(4 * L);
#if PY_VERSION_HEX >= 0x030D0000
    if (_PyLong_AsByteArray((PyLongObject*)v, dst, (size_t)(4 * L), 1, 1, 1) < 0) return 0;
#else
    if (_PyLong_AsByteArray((PyLongObject*)v, dst, (size_t)(4 * L), 1, 1) < 0) return 0;
#endif
  }
  return 1;
}

static PyObject* lead_row(PyObject* terms, int swap, long row, int16_t deg) {
  PyObject* out = PyList_New(deg + 1);
  if (!out) return NULL;
  PyObject* zero = PyLong_FromLong(0);
  for (Py_ssize_t t = 0; t <= deg; ++t) {
    Py_INCREF(zero);
    PyList_SET_ITEM(out, t, zero);
  }
  Py_DECREF(zero);
  Py_ssize_t pos = 0;
  PyObject *k, *v;
  long i, j;
  while (PyDict_Next(terms, &pos, &k, &v)) {
    key_ij(k, swap, &i, &j);
    if (j != row || _PyLong_Sign(v) == 0) continue;
    Py_INCREF(v);
    PyList_SetItem(out, i, v); /* steals v, releases the zero */
  }
  return out;
}

static PyObject* norms_list(const GridSide* f, const GridSide* g) {
  if (!f->norm_ok || !g->norm_ok) Py_RETURN_NONE;
  PyObject* out = PyList_New(f->rows + g->rows);
  if (!out) return NULL;
  for (Py_ssize_t r = 0; r < f->rows; ++r) PyList_SET_ITEM(out, r, PyFloat_FromDouble(f->norm[r]));
  for (Py_ssize_t r = 0; r < g->rows; ++r) PyList_SET_ITEM(out, f->rows + r, PyFloat_FromDouble(g->norm[r]));
  return out;
}

static PyObject* terms_grid(PyObject* self, PyObject* args) {
  PyObject *tf, *tg;
  int swap;
  if (!PyArg_ParseTuple(args, "OOp", &tf, &tg, &swap)) return NULL;
  if (!PyDict_CheckExact(tf) || !PyDict_CheckExact(tg)) Py_RETURN_NONE;
  GridSide f = {0}, g = {0};
  size_t maxbits = 0;
  PyObject* ret = NULL;
  int okf = scan_side(tf, swap, &f, &maxbits);
  int okg = okf == 1 ? scan_side(tg, swap, &g, &maxbits) : okf;
  if (okf < 0 || okg < 0) {
    PyErr_NoMemory();
    goto done;
  }
  if (!okf || !okg || f.rows == 0 || g.rows == 0) {
    Py_INCREF(Py_None);
    ret = Py_None;
    goto done;
  }
  {
    const Py_ssize_t L = (Py_ssize_t)((maxbits + 1 + 31) / 32) > 0 ? (Py_ssize_t)((maxbits + 1 + 31) / 32) : 1;
    const Py_ssize_t cf = f.rows * (f.dx + 1), C = cf + g.rows * (g.dx + 1);
    PyObject* limbs = PyBytes_FromStringAndSize(NULL, C * L * 4);
    if (!limbs) goto done;
    unsigned char* buf = (unsigned char*)PyBytes_AS_STRING(limbs);
    memset(buf, 0, (size_t)(C * L * 4));
    if (!write_side(tf, swap, f.dx, L, buf) || !write_side(tg, swap, g.dx, L, buf + (size_t)cf * L * 4)) {
      Py_DECREF(limbs);
      goto done;
    }
    PyObject* degs = PyBytes_FromStringAndSize(NULL, (f.rows + g.rows) * 2);
    if (!degs) {
      Py_DECREF(limbs);
      goto done;
    }
    memcpy(PyBytes_AS_STRING(degs), f.deg, (size_t)f.rows * 2);
    memcpy(PyBytes_AS_STRING(degs) + f.rows * 2, g.deg, (size_t)g.rows * 2);
    PyObject* norms = norms_list(&f, &g);
    PyObject* lcf = lead_row(tf, swap, (long)(f.rows - 1), f.deg[f.rows - 1]);
    PyObject* lcg = lead_row(tg, swap, (long)(g.rows - 1), g.deg[g.rows - 1]);
    if (norms && lcf && lcg)
      ret = Py_BuildValue("(NnnnnnllNNNN)", limbs, L, f.rows - 1, g.rows - 1, f.dx, g.dx, f.td, g.td, degs, norms,
                          lcf, lcg);
    else {
      Py_DECREF(limbs);
      Py_DECREF(degs);
      Py_XDECREF(norms);
      Py_XDECREF(lcf);
      Py_XDECREF(lcg);
    }
  }
done:
  PyMem_Free(f.deg);
  PyMem_Free(f.norm);
  PyMem_Free(g.deg);
  PyMem_Free(g.norm);
  return ret;
}

/* [c mod p for c in ints] for a word prime p < 2^32 (the single-prime residues of
 * modular_subres_profile, modpoly.py:437-438): Horner over CPython's 30-bit digits
 * with a 64-bit reciprocal (~0.4 ns per digit; Python's % takes the general long
 * division for a two-digit divisor: ~2.4 us per 5,000-bit coefficient). */
static PyObject* mod_list(PyObject* self, PyObject* args) {
  PyObject* lst;
  unsigned long long pl;
  if (!PyArg_ParseTuple(args, "OK", &lst, &pl)) return NULL;
  if (pl < 2 || pl >= (1ull << 32)) {
    PyErr_SetString(PyExc_ValueError, "mod_list: need 2 <= p < 2^32");
    return NULL;
  }
  PyObject* seq = PySequence_Fast(lst, "mod_list: expected a sequence of ints");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  PyObject** items = PySequence_Fast_ITEMS(seq);
  PyObject* out = PyList_New(n);
  if (!out) {
    Py_DECREF(seq);
    return NULL;
  }
  const uint64_t p = (uint64_t)pl, m = ~0ull / p;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* v = items[i];
    if (!PyLong_Check(v)) {
      Py_DECREF(seq);
      Py_DECREF(out);
      PyErr_SetString(PyExc_TypeError, "mod_list: expected ints");
      return NULL;
    }
    uint64_t r = 0;
#ifdef CKB_FAST_DIGITS
    const uintptr_t tag = ((PyLongObject*)v)->long_value.lv_tag;
    const Py_ssize_t nd = (Py_ssize_t)(tag >> 3);
    const int neg = (tag & 3) == 2;
    const digit* d = ((PyLongObject*)v)->long_value.ob_digit;
    for (Py_ssize_t k = nd - 1; k >= 0; --k) {
      const uint64_t x = (r << PyLong_SHIFT) | (uint64_t)d[k];  /* < p 2^30 < 2^62 */
      const uint64_t q = (uint64_t)(((unsigned __int128)x * m) >> 64);
      r = x - q * p;
      while (r >= p) r -= p;
    }
#else
    PyObject* pr = PyLong_FromUnsignedLongLong(pl);
    PyObject* rm = PyNumber_Remainder(v, pr);
    Py_DECREF(pr);
    if (!rm) {
      Py_DECREF(seq);
      Py_DECREF(out);
      return NULL;
    }
    r = PyLong_AsUnsignedLongLong(rm);
    Py_DECREF(rm);
    const int neg = 0;
#endif
    if (neg && r) r = p - r;
    PyList_SET_ITEM(out, i, PyLong_FromUnsignedLongLong(r));
  }
  Py_DECREF(seq);
  return out;
}

static PyMethodDef methods[] = {
    {"mod_list", mod_list, METH_VARARGS, "(ints, p) -> [c mod p for c in ints] (canonical residues)"},
    {"limbs_to_ints", limbs_to_ints, METH_VARARGS, "[N][LW] two's-complement u32 limbs -> list of ints"},
    {"terms_grid", terms_grid, METH_VARARGS,
     "(terms_f, terms_g, swap) -> packed limb grid, shape, degrees, row 1-norms, leading rows (or None)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "ckb_limbs", NULL, -1, methods};

PyMODINIT_FUNC PyInit_ckb_limbs(void) { return PyModule_Create(&mod); }
