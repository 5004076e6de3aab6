/* Host-side conversion of the engine's output limbs to Python ints.
 *
 * The reference returns list[int] (modpoly.py:348-394); the device writes each
 * coefficient as LW two's-complement little-endian 32-bit limbs.  This builds
 * the list in one C loop, dropping sign-extension limbs first so small
 * coefficients convert in proportion to their size.  (Python-API glue, not
 * part of the compute path.) */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#if PY_VERSION_HEX >= 0x030C0000 && PY_VERSION_HEX < 0x030E0000 && PyLong_SHIFT == 30
#define CKB_FAST_DIGITS 1
/* Magnitude of a two's-complement limb array repacked straight into CPython's
 * 30-bit digits (_PyLong_FromDigits copies and normalises them): O(limbs),
 * no per-byte loop (_PyLong_FromByteArray costs ~1 us per 5,000-bit
 * coefficient; this ~0.1 us). */
/* digit of the magnitude at bit offset `bit` (bounds-checked) */
static inline digit digit_at(const uint32_t* a, Py_ssize_t len, Py_ssize_t bit) {
  const Py_ssize_t w = bit >> 5;
  const int o = (int)(bit & 31);
  uint64_t v = (uint64_t)a[w] >> o;
  if (w + 1 < len) v |= (uint64_t)a[w + 1] << (32 - o);
  return (digit)(v & PyLong_MASK);
}

/* the magnitude's digits into dg (room for len * 32 / 30 + 2), returns the
 * normalised digit count; *neg = sign; mag: scratch of len + 2 words (no
 * Python API: runs without the GIL).  Each digit is one unaligned 64-bit load,
 * a shift and a mask; a negative value's magnitude (~c + 1: zero below the
 * lowest nonzero limb, its negation there, ~c above -- no carry chain) is
 * formed in the scratch first. */
static Py_ssize_t limbs_to_digits(const uint32_t* c, Py_ssize_t len, digit* dg, int* negp, uint32_t* mag) {
  const int neg = (int)(c[len - 1] >> 31);
  const uint32_t* src = c;
  if (neg) {
    Py_ssize_t f = 0;
    while (c[f] == 0u) ++f; /* a negative value has a nonzero limb */
    for (Py_ssize_t k = 0; k < f; ++k) mag[k] = 0u;
    mag[f] = 0u - c[f];
    for (Py_ssize_t k = f + 1; k < len; ++k) mag[k] = ~c[k];
    mag[len] = 0u;
    mag[len + 1] = 0u;
    src = mag;
  }
  const Py_ssize_t nd0 = (len * 32 + PyLong_SHIFT - 1) / PyLong_SHIFT;
  /* digits whose 8-byte window lies inside the limbs (all of them with the padded scratch) */
  const Py_ssize_t lim = neg ? 4 * len + 8 : 4 * len;
  const unsigned char* bytes = (const unsigned char*)src;
  /* four digits = 120 bits = 15 bytes: windows at byte offsets 0, 3, 7, 11 of
   * each 15-byte group, shifted by 0, 6, 4, 2 bits (PyLong_SHIFT == 30) */
  Py_ssize_t q = 0;
  const Py_ssize_t nq = nd0 / 4;
  for (; q < nq && 15 * q + 11 + 8 <= lim; ++q) {
    const unsigned char* g = bytes + 15 * q;
    uint64_t x0, x1, x2, x3;
    memcpy(&x0, g, 8);
    memcpy(&x1, g + 3, 8);
    memcpy(&x2, g + 7, 8);
    memcpy(&x3, g + 11, 8);
    digit* d = dg + 4 * q;
    d[0] = (digit)(x0 & PyLong_MASK);
    d[1] = (digit)((x1 >> 6) & PyLong_MASK);
    d[2] = (digit)((x2 >> 4) & PyLong_MASK);
    d[3] = (digit)((x3 >> 2) & PyLong_MASK);
  }
  for (Py_ssize_t t = 4 * q; t < nd0; ++t) dg[t] = digit_at(src, len, (Py_ssize_t)PyLong_SHIFT * t);
  Py_ssize_t nd = nd0;
  while (nd > 0 && dg[nd - 1] == 0) --nd;
  *negp = neg;
  return nd;
}
#endif

/* Pass 2 of limbs_to_ints can be split with one persistent helper thread (created
 * on first use of a large result, parked on a condition variable): the caller
 * fills the first half of the coefficients, the helper the second.
 * CKB_CONVERT_THREADS=0 disables it; it is also skipped for results under 4 MB and
 * on hosts with fewer than 4 CPUs. */
#include <pthread.h>
#include <sched.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <unistd.h>
typedef struct {
  const uint32_t* w;
  Py_ssize_t lw, k0, k1;
  const Py_ssize_t* lens;
  PyObject** items;
  uint32_t* mag;
} FillJob;
static void fill_range(const FillJob* j) {
  for (Py_ssize_t k = j->k0; k < j->k1; ++k) {
    if (!j->lens[k]) continue;
    PyLongObject* v = (PyLongObject*)j->items[k];
    int neg = 0;
    const Py_ssize_t nd = limbs_to_digits(j->w + k * j->lw, j->lens[k], v->long_value.ob_digit, &neg, j->mag);
    /* lv_tag = digit count << 3 | sign (0: positive, 1: zero, 2: negative) */
    v->long_value.lv_tag = nd ? ((uintptr_t)nd << 3) | (neg ? 2u : 0u) : 1u;
    if (!nd) v->long_value.ob_digit[0] = 0;
  }
}
static pthread_mutex_t g_fill_mu = PTHREAD_MUTEX_INITIALIZER;
static pthread_cond_t g_fill_cv = PTHREAD_COND_INITIALIZER;
static FillJob g_fill_job;
static int g_fill_has = 0;
static atomic_int g_fill_done;
static int g_fill_state = -1; /* -1 unknown, 0 off, 1 helper running */
static void* fill_worker(void* arg) {
  (void)arg;
  for (;;) {
    pthread_mutex_lock(&g_fill_mu);
    while (!g_fill_has) pthread_cond_wait(&g_fill_cv, &g_fill_mu);
    FillJob j = g_fill_job;
    g_fill_has = 0;
    pthread_mutex_unlock(&g_fill_mu);
    fill_range(&j);
    atomic_store_explicit(&g_fill_done, 1, memory_order_release);
  }
  return NULL;
}
/* a forked child has no helper thread: start over there */
static void fill_atfork_child(void) {
  pthread_mutex_t m = PTHREAD_MUTEX_INITIALIZER;
  pthread_cond_t c = PTHREAD_COND_INITIALIZER;
  g_fill_mu = m;
  g_fill_cv = c;
  g_fill_has = 0;
  g_fill_state = -1;
}
static int fill_helper_ready(void) {
  if (g_fill_state < 0) {
    static int atfork = 0;
    if (!atfork) {
      pthread_atfork(NULL, NULL, fill_atfork_child);
      atfork = 1;
    }
    const char* e = getenv("CKB_CONVERT_THREADS");
    long ncpu = sysconf(_SC_NPROCESSORS_ONLN);
    g_fill_state = 0;
    if (!(e && e[0] == '0') && ncpu >= 4) {
      pthread_t t;
      pthread_attr_t at;
      pthread_attr_init(&at);
      pthread_attr_setdetachstate(&at, PTHREAD_CREATE_DETACHED);
      if (pthread_create(&t, &at, fill_worker, NULL) == 0) g_fill_state = 1;
      pthread_attr_destroy(&at);
    }
  }
  return g_fill_state == 1;
}

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
  uint32_t* mag = (uint32_t*)PyMem_RawMalloc(sizeof(uint32_t) * (size_t)(lw + 2));
  if (!mag) {
    PyMem_Free(lens);
    Py_DECREF(out);
    PyBuffer_Release(&view);
    return PyErr_NoMemory();
  }
  /* the helper gets the second half only for large results (>= 1 M limbs, 4 MB: cfg5's
   * 36 MB result converts in 2.1 ms instead of 8.6 ms); below that the wake-up and the
   * CPU-quota cost on the next call outweigh it (cfg4, 1.1 MB: 0.18 ms alone, 0.19-0.21 split) */
  const int split = (Py_ssize_t)n * lw >= ((Py_ssize_t)1 << 20) && fill_helper_ready();
  uint32_t* mag2 = split ? (uint32_t*)PyMem_RawMalloc(sizeof(uint32_t) * (size_t)(lw + 2)) : NULL;
  Py_BEGIN_ALLOW_THREADS
  FillJob mine = {w, lw, 0, n, lens, items, mag};
  if (mag2) {
    const Py_ssize_t h = n / 2;
    FillJob theirs = {w, lw, h, n, lens, items, mag2};
    mine.k1 = h;
    atomic_store_explicit(&g_fill_done, 0, memory_order_relaxed);
    pthread_mutex_lock(&g_fill_mu);
    g_fill_job = theirs;
    g_fill_has = 1;
    pthread_cond_signal(&g_fill_cv);
    pthread_mutex_unlock(&g_fill_mu);
  }
  fill_range(&mine);
  if (mag2)
    while (!atomic_load_explicit(&g_fill_done, memory_order_acquire)) sched_yield();
  Py_END_ALLOW_THREADS
  if (mag2) PyMem_RawFree(mag2);
  PyMem_RawFree(mag);
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

/* one term: borrowed coefficient (the dicts outlive the call), exponents */
typedef struct {
  PyObject* v;
  int32_t i, j;
} Ent;

/* small non-negative int (an exponent); 0 = not a plain int in range */
static int small_exp(PyObject* o, long* x) {
  if (!PyLong_CheckExact(o)) return 0;
#if PY_VERSION_HEX >= 0x030C0000
  if (PyUnstable_Long_IsCompact((PyLongObject*)o)) {
    *x = (long)PyUnstable_Long_CompactValue((PyLongObject*)o);
    return *x >= 0 && *x <= 1000000;
  }
  return 0;
#else
  *x = PyLong_AsLong(o);
  if (*x == -1 && PyErr_Occurred()) {
    PyErr_Clear();
    return 0;
  }
  return *x >= 0 && *x <= 1000000;
#endif
}

/* pass 1 (the only walk of the dict): nonzero terms into an array with shape,
 * degrees, 1-norms and the widest coefficient; 0 = not plain, -1 = no memory */
static int scan_side(PyObject* terms, int swap, GridSide* s, size_t* maxbits, Ent** ents, Py_ssize_t* nent) {
  Py_ssize_t pos = 0, n = 0;
  PyObject *k, *v;
  long i, j, maxj = -1, maxi = -1;
  s->td = -1;
  Ent* e = (Ent*)PyMem_Malloc(sizeof(Ent) * (size_t)(PyDict_GET_SIZE(terms) + 1));
  if (!e) return -1;
  *ents = e;
  while (PyDict_Next(terms, &pos, &k, &v)) {
    if (!PyLong_CheckExact(v) || !PyTuple_CheckExact(k) || PyTuple_GET_SIZE(k) != 2) return 0;
    long a, b;
    if (!small_exp(PyTuple_GET_ITEM(k, 0), &a) || !small_exp(PyTuple_GET_ITEM(k, 1), &b)) return 0;
    if (_PyLong_Sign(v) == 0) continue;
    i = swap ? b : a;
    j = swap ? a : b;
    e[n].v = v;
    e[n].i = (int32_t)i;
    e[n].j = (int32_t)j;
    ++n;
    if (j > maxj) maxj = j;
    if (i > maxi) maxi = i;
    if (i + j > s->td) s->td = i + j;
  }
  *nent = n;
  s->rows = maxj + 1;
  s->dx = maxi < 0 ? 0 : maxi;
  s->deg = (int16_t*)PyMem_Malloc(sizeof(int16_t) * (size_t)(s->rows > 0 ? s->rows : 1));
  s->norm = (double*)PyMem_Calloc((size_t)(s->rows > 0 ? s->rows : 1), sizeof(double));
  if (!s->deg || !s->norm) return -1;
  for (Py_ssize_t r = 0; r < s->rows; ++r) s->deg[r] = -1;
  s->norm_ok = 1;
  for (Py_ssize_t t = 0; t < n; ++t) {
    const int32_t ti = e[t].i, tj = e[t].j;
    if (ti > s->deg[tj]) s->deg[tj] = (int16_t)ti;
    const size_t nb = _PyLong_NumBits(e[t].v);
    if (nb > *maxbits) *maxbits = nb;
    if (s->norm_ok) {
      const double d = PyLong_AsDouble(e[t].v);
      if (d == -1.0 && PyErr_Occurred()) {
        PyErr_Clear();
        s->norm_ok = 0;
      } else {
        s->norm[tj] += d < 0 ? -d : d;
      }
    }
  }
  return 1;
}

/* one coefficient as L two's-complement little-endian u32 limbs (dst zeroed;
 * the caller sized L for the widest magnitude plus a sign bit) */
static int put_limbs(PyObject* v, unsigned char* dst, Py_ssize_t L) {
#ifdef CKB_FAST_DIGITS
  const uintptr_t tag = ((PyLongObject*)v)->long_value.lv_tag;
  const Py_ssize_t nd = (Py_ssize_t)(tag >> 3);
  const int neg = (tag & 3) == 2;
  const digit* d = ((PyLongObject*)v)->long_value.ob_digit;
  uint32_t* w = (uint32_t*)dst;
  uint64_t acc = 0;
  int bits = 0;
  Py_ssize_t k = 0;
  for (Py_ssize_t t = 0; t < nd; ++t) {
    acc |= (uint64_t)d[t] << bits;
    bits += PyLong_SHIFT;
    if (bits >= 32) {
      if (k < L) w[k] = (uint32_t)acc;
      ++k;
      acc >>= 32;
      bits -= 32;
    }
  }
  if (bits > 0 && k < L) w[k] = (uint32_t)acc;
  if (neg) { /* two's complement: invert, add one */
    uint64_t cy = 1;
    for (Py_ssize_t t = 0; t < L; ++t) {
      const uint64_t x = (uint64_t)(uint32_t)~w[t] + cy;
      w[t] = (uint32_t)x;
      cy = x >> 32;
    }
  }
  return 1;
#elif PY_VERSION_HEX >= 0x030D0000
  return _PyLong_AsByteArray((PyLongObject*)v, dst, (size_t)(4 * L), 1, 1, 1) >= 0;
#else
  return _PyLong_AsByteArray((PyLongObject*)v, dst, (size_t)(4 * L), 1, 1) >= 0;
#endif
}

/* pass 2: every nonzero coefficient into its grid slot */
static int write_side(const Ent* e, Py_ssize_t n, Py_ssize_t dx, Py_ssize_t L, unsigned char* base) {
  for (Py_ssize_t t = 0; t < n; ++t) {
    unsigned char* dst = base + ((size_t)e[t].j * (size_t)(dx + 1) + (size_t)e[t].i) * (size_t)(4 * L);
    if (!put_limbs(e[t].v, dst, L)) return 0;
  }
  return 1;
}

static PyObject* lead_row(const Ent* e, Py_ssize_t n, long row, int16_t deg) {
  PyObject* out = PyList_New(deg + 1);
  if (!out) return NULL;
  PyObject* zero = PyLong_FromLong(0);
  for (Py_ssize_t t = 0; t <= deg; ++t) {
    Py_INCREF(zero);
    PyList_SET_ITEM(out, t, zero);
  }
  Py_DECREF(zero);
  for (Py_ssize_t t = 0; t < n; ++t) {
    if (e[t].j != row) continue;
    Py_INCREF(e[t].v);
    PyList_SetItem(out, e[t].i, e[t].v); /* steals v, releases the zero */
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
  Ent *ef = NULL, *eg = NULL;
  Py_ssize_t nf = 0, ng = 0;
  size_t maxbits = 0;
  PyObject* ret = NULL;
  int okf = scan_side(tf, swap, &f, &maxbits, &ef, &nf);
  int okg = okf == 1 ? scan_side(tg, swap, &g, &maxbits, &eg, &ng) : okf;
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
    if (!write_side(ef, nf, f.dx, L, buf) || !write_side(eg, ng, g.dx, L, buf + (size_t)cf * L * 4)) {
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
    PyObject* lcf = lead_row(ef, nf, (long)(f.rows - 1), f.deg[f.rows - 1]);
    PyObject* lcg = lead_row(eg, ng, (long)(g.rows - 1), g.deg[g.rows - 1]);
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
  PyMem_Free(ef);
  PyMem_Free(eg);
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

/* planner.log2_bound_from_norms in one C pass (host planning of every call):
 * the reference's column-sum bound, the Hadamard column bound and the row
 * bound of the Sylvester matrix from the per-row 1-norms (doubles); window
 * sums taken directly (all terms positive, no prefix-sum cancellation). */
static PyObject* norms_log2_bound(PyObject* self, PyObject* args) {
  PyObject *af, *ag;
  if (!PyArg_ParseTuple(args, "OO", &af, &ag)) return NULL;
  PyObject* sf = PySequence_Fast(af, "norms_log2_bound: expected sequences of floats");
  if (!sf) return NULL;
  PyObject* sg = PySequence_Fast(ag, "norms_log2_bound: expected sequences of floats");
  if (!sg) {
    Py_DECREF(sf);
    return NULL;
  }
  const Py_ssize_t lf = PySequence_Fast_GET_SIZE(sf), lg = PySequence_Fast_GET_SIZE(sg);
  double* v = (double*)PyMem_Malloc(sizeof(double) * (size_t)(lf + lg + 1));
  PyObject* ret = NULL;
  if (!v) {
    PyErr_NoMemory();
    goto out;
  }
  for (Py_ssize_t i = 0; i < lf + lg; ++i) {
    PyObject* o = i < lf ? PySequence_Fast_GET_ITEM(sf, i) : PySequence_Fast_GET_ITEM(sg, i - lf);
    v[i] = PyFloat_AsDouble(o);
    if (v[i] == -1.0 && PyErr_Occurred()) goto out;
  }
  {
    const double* nf = v;
    const double* ng = v + lf;
    const Py_ssize_t m = lf - 1, n = lg - 1; /* y-degrees */
    double ref = 0.0, col = 0.0, sf2 = 0.0, sg2 = 0.0;
    for (Py_ssize_t i = 0; i <= m; ++i) sf2 += nf[i] * nf[i];
    for (Py_ssize_t i = 0; i <= n; ++i) sg2 += ng[i] * ng[i];
    /* column t (0 <= t < m + n): f rows i with t - n < i <= t, g rows with t - m < i <= t */
    for (Py_ssize_t t = 0; t < m + n; ++t) {
      double s1 = 0.0, s2 = 0.0;
      for (Py_ssize_t i = (t - n + 1 > 0 ? t - n + 1 : 0); i <= t && i <= m; ++i) {
        s1 += nf[i];
        s2 += nf[i] * nf[i];
      }
      for (Py_ssize_t i = (t - m + 1 > 0 ? t - m + 1 : 0); i <= t && i <= n; ++i) {
        s1 += ng[i];
        s2 += ng[i] * ng[i];
      }
      ref += log2(s1 > 1.0 ? s1 : 1.0);
      col += 0.5 * log2(s2 > 1.0 ? s2 : 1.0);
    }
    const double row = 0.5 * ((double)n * log2(sf2 > 1.0 ? sf2 : 1.0) + (double)m * log2(sg2 > 1.0 ? sg2 : 1.0));
    double b = ref < row ? ref : row;
    if (col < b) b = col;
    ret = PyFloat_FromDouble(b);
  }
out:
  PyMem_Free(v);
  Py_DECREF(sf);
  Py_DECREF(sg);
  return ret;
}

static PyMethodDef methods[] = {
    {"norms_log2_bound", norms_log2_bound, METH_VARARGS,
     "(norms_f, norms_g) -> log2 of the Sylvester coefficient bound from the per-row 1-norms"},
    {"mod_list", mod_list, METH_VARARGS, "(ints, p) -> [c mod p for c in ints] (canonical residues)"},
    {"limbs_to_ints", limbs_to_ints, METH_VARARGS, "[N][LW] two's-complement u32 limbs -> list of ints"},
    {"terms_grid", terms_grid, METH_VARARGS,
     "(terms_f, terms_g, swap) -> packed limb grid, shape, degrees, row 1-norms, leading rows (or None)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef mod = {PyModuleDef_HEAD_INIT, "ckb_limbs", NULL, -1, methods};

PyMODINIT_FUNC PyInit_ckb_limbs(void) { return PyModule_Create(&mod); }
