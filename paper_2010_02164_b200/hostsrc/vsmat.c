/* _vsmat: bulk materialisation of decode outputs as Candidate objects.
 *
 * The reference API returns list[list[Candidate]] (bb/scheduler.py:287,
 * bb/core.py:50-61).  Building ~10^5 frozen-dataclass objects in Python costs
 * more than the device decode itself, so the host runtime builds them here:
 * each Candidate is allocated with its type's tp_alloc and its four __slots__
 * are filled directly (the member offsets are read from the class's slot
 * descriptors), tokens become a tuple of ints.  Pure host bookkeeping, no
 * search arithmetic.
 *
 *   fill(out, gids, lo, count, lens, scores, offs, toks, k, Candidate)
 *     out     list, out[g] is replaced for every input g of the chunk
 *     gids    int64 array (local -> global input id) or None (identity)
 *     lo      first local input of the chunk
 *     count   int32[nq]      candidates emitted per input of the chunk
 *     lens    int32[nq*k]    per-candidate token counts
 *     scores  float64[nq*k]  fp64 scores
 *     offs    int32[nq*k]    start of each candidate's tokens in toks
 *     toks    int32[*]       the host copy of out_tok (absolute offsets)
 *     k = 0: lens/scores/offs hold only the emitted candidates, consecutive
 *
 *   fill_packed(out, gids, count, lens, scores, toks, Candidate)
 *     the packed layout of the multi-GPU gather: each input's candidates are
 *     consecutive in lens/scores and their tokens consecutive in toks
 *
 *   flatten(corpus, V) -> (tok bytearray int32[total], off bytearray int32[N+1], ok)
 *     the corpus (a sequence of token sequences) flattened in one C pass for
 *     the device upload; ok = 0 when an input is empty or a token is outside
 *     [0, V) (the caller re-checks to raise the reference's DataError); None
 *     when an item is not a sequence of ints (the caller's generic path)
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>

static Py_ssize_t slot_offset(PyObject* type, const char* name) {
  PyObject* d = PyObject_GetAttrString(type, name);
  if (!d) return -1;
  Py_ssize_t off = -1;
  if (Py_IS_TYPE(d, &PyMemberDescr_Type)) off = ((PyMemberDescrObject*)d)->d_member->offset;
  Py_DECREF(d);
  if (off < 0) PyErr_Format(PyExc_TypeError, "%s is not a __slots__ member", name);
  return off;
}

/* Token ids repeat across candidates: one cached int object per id (grown on
 * demand), so a token tuple costs increfs instead of allocations. */
static PyObject** tok_cache = NULL;
static Py_ssize_t tok_cache_n = 0;

static inline PyObject* tok_obj(int32_t t) {
  if (t >= 0 && t < tok_cache_n) {
    PyObject* o = tok_cache[t];
    Py_INCREF(o);
    return o;
  }
  return PyLong_FromLong(t);
}

static int grow_cache(Py_ssize_t want) {
  if (want <= tok_cache_n || want > (1 << 24)) return 0;
  PyObject** c = (PyObject**)PyMem_Realloc(tok_cache, want * sizeof(PyObject*));
  if (!c) return -1;
  tok_cache = c;
  for (Py_ssize_t i = tok_cache_n; i < want; ++i) {
    c[i] = PyLong_FromSsize_t(i);
    if (!c[i]) return -1;
    tok_cache_n = i + 1;
  }
  return 0;
}

/* reserve(V): cache the int objects of token ids [0, V) */
static PyObject* reserve(PyObject* self, PyObject* args) {
  Py_ssize_t v;
  if (!PyArg_ParseTuple(args, "n", &v)) return NULL;
  if (grow_cache(v) < 0) return PyErr_NoMemory();
  Py_RETURN_NONE;
}

static inline void set_slot(PyObject* obj, Py_ssize_t off, PyObject* v) {
  PyObject** p = (PyObject**)((char*)obj + off);
  PyObject* old = *p;
  *p = v; /* steals v */
  Py_XDECREF(old);
}

static PyObject* fill(PyObject* self, PyObject* args) {
  PyObject *out, *gids_o, *type;
  Py_ssize_t lo, k;
  Py_buffer count, lens, scores, offs, toks, gids = {0};
  if (!PyArg_ParseTuple(args, "O!Ony*y*y*y*y*nO", &PyList_Type, &out, &gids_o, &lo, &count, &lens, &scores,
                        &offs, &toks, &k, &type))
    return NULL;
  PyObject* ret = NULL;
  const int has_gids = gids_o != Py_None;
  if (has_gids && PyObject_GetBuffer(gids_o, &gids, PyBUF_SIMPLE) < 0) goto done;
  Py_ssize_t o_tok = slot_offset(type, "tokens"), o_sc = slot_offset(type, "score"),
             o_fin = slot_offset(type, "finalized"), o_in = slot_offset(type, "input_id");
  if (o_tok < 0 || o_sc < 0 || o_fin < 0 || o_in < 0) goto done;
  if (!PyType_Check(type)) {
    PyErr_SetString(PyExc_TypeError, "Candidate type expected");
    goto done;
  }
  PyTypeObject* tp = (PyTypeObject*)type;
  const int32_t* cnt = (const int32_t*)count.buf;
  const int32_t* ln = (const int32_t*)lens.buf;
  const double* sc = (const double*)scores.buf;
  const int32_t* of = (const int32_t*)offs.buf;
  const int32_t* tk = (const int32_t*)toks.buf;
  const Py_ssize_t ntok = toks.len / 4, nq = count.len / 4, nout = PyList_GET_SIZE(out), ne = lens.len / 4;
  Py_ssize_t run = 0;
  for (Py_ssize_t q = 0; q < nq; ++q) {
    const long long gi = has_gids ? ((const long long*)gids.buf)[lo + q] : (long long)(lo + q);
    if (gi < 0 || gi >= nout) {
      PyErr_SetString(PyExc_IndexError, "input id outside the output list");
      goto done;
    }
    const int c = cnt[q];
    if (c < 0 || (k > 0 && c > k) || (k == 0 && run + c > ne) || (k > 0 && (q + 1) * k > ne)) {
      PyErr_SetString(PyExc_ValueError, "bad candidate count");
      goto done;
    }
    PyObject* per = PyList_New(c);
    if (!per) goto done;
    for (int e = 0; e < c; ++e) {
      const Py_ssize_t j = k > 0 ? q * k + e : run++;  /* k == 0: compacted, consecutive */
      const Py_ssize_t b = of[j], n = ln[j];
      if (n < 0 || b < 0 || b + n > ntok) {
        Py_DECREF(per);
        PyErr_SetString(PyExc_ValueError, "candidate tokens outside the token buffer");
        goto done;
      }
      PyObject* tup = PyTuple_New(n);
      if (!tup) {
        Py_DECREF(per);
        goto done;
      }
      for (Py_ssize_t p = 0; p < n; ++p) PyTuple_SET_ITEM(tup, p, tok_obj(tk[b + p]));
      PyObject* cand = tp->tp_alloc(tp, 0);
      if (!cand) {
        Py_DECREF(tup);
        Py_DECREF(per);
        goto done;
      }
      set_slot(cand, o_tok, tup);
      set_slot(cand, o_sc, PyFloat_FromDouble(sc[j]));
      Py_INCREF(Py_True);
      set_slot(cand, o_fin, Py_True);
      set_slot(cand, o_in, PyLong_FromLongLong(gi));
      PyList_SET_ITEM(per, e, cand);
    }
    if (PyList_SetItem(out, (Py_ssize_t)gi, per) < 0) goto done; /* steals per */
  }
  ret = Py_None;
  Py_INCREF(ret);
done:
  if (has_gids && gids.buf) PyBuffer_Release(&gids);
  PyBuffer_Release(&count);
  PyBuffer_Release(&lens);
  PyBuffer_Release(&scores);
  PyBuffer_Release(&offs);
  PyBuffer_Release(&toks);
  return ret;
}

static PyObject* fill_packed(PyObject* self, PyObject* args) {
  PyObject *out, *gids_o, *type;
  Py_buffer gids, count, lens, scores, toks;
  if (!PyArg_ParseTuple(args, "O!y*y*y*y*y*O", &PyList_Type, &out, &gids, &count, &lens, &scores, &toks, &type))
    return NULL;
  (void)gids_o;
  PyObject* ret = NULL;
  Py_ssize_t o_tok = slot_offset(type, "tokens"), o_sc = slot_offset(type, "score"),
             o_fin = slot_offset(type, "finalized"), o_in = slot_offset(type, "input_id");
  if (o_tok < 0 || o_sc < 0 || o_fin < 0 || o_in < 0) goto done;
  PyTypeObject* tp = (PyTypeObject*)type;
  const long long* gi_ = (const long long*)gids.buf;
  const int32_t* cnt = (const int32_t*)count.buf;
  const int32_t* ln = (const int32_t*)lens.buf;
  const double* sc = (const double*)scores.buf;
  const int32_t* tk = (const int32_t*)toks.buf;
  const Py_ssize_t nq = count.len / 4, ne = lens.len / 4, ntok = toks.len / 4, nout = PyList_GET_SIZE(out);
  if (gids.len / 8 < nq) {
    PyErr_SetString(PyExc_ValueError, "fewer ids than inputs");
    goto done;
  }
  Py_ssize_t e = 0, t = 0;
  for (Py_ssize_t q = 0; q < nq; ++q) {
    const long long gi = gi_[q];
    const int c = cnt[q];
    if (gi < 0 || gi >= nout || c < 0 || e + c > ne) {
      PyErr_SetString(PyExc_ValueError, "packed results inconsistent");
      goto done;
    }
    PyObject* per = PyList_New(c);
    if (!per) goto done;
    for (int i = 0; i < c; ++i, ++e) {
      const Py_ssize_t n = ln[e];
      if (n < 0 || t + n > ntok) {
        Py_DECREF(per);
        PyErr_SetString(PyExc_ValueError, "packed tokens inconsistent");
        goto done;
      }
      PyObject* tup = PyTuple_New(n);
      if (!tup) {
        Py_DECREF(per);
        goto done;
      }
      for (Py_ssize_t p = 0; p < n; ++p) PyTuple_SET_ITEM(tup, p, tok_obj(tk[t + p]));
      t += n;
      PyObject* cand = tp->tp_alloc(tp, 0);
      if (!cand) {
        Py_DECREF(tup);
        Py_DECREF(per);
        goto done;
      }
      set_slot(cand, o_tok, tup);
      set_slot(cand, o_sc, PyFloat_FromDouble(sc[e]));
      Py_INCREF(Py_True);
      set_slot(cand, o_fin, Py_True);
      set_slot(cand, o_in, PyLong_FromLongLong(gi));
      PyList_SET_ITEM(per, i, cand);
    }
    if (PyList_SetItem(out, (Py_ssize_t)gi, per) < 0) goto done;
  }
  ret = Py_None;
  Py_INCREF(ret);
done:
  PyBuffer_Release(&gids);
  PyBuffer_Release(&count);
  PyBuffer_Release(&lens);
  PyBuffer_Release(&scores);
  PyBuffer_Release(&toks);
  return ret;
}

static PyObject* flatten(PyObject* self, PyObject* args) {
  PyObject* corpus;
  long long V;
  if (!PyArg_ParseTuple(args, "OL", &corpus, &V)) return NULL;
  PyObject* seq = PySequence_Fast(corpus, "corpus must be a sequence");
  if (!seq) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(seq);
  PyObject** items = PySequence_Fast_ITEMS(seq);
  PyObject *off = NULL, *tok = NULL, *ret = NULL;
  off = PyByteArray_FromStringAndSize(NULL, (n + 1) * (Py_ssize_t)sizeof(int32_t));
  if (!off) goto done;
  int32_t* po = (int32_t*)PyByteArray_AS_STRING(off);
  long long total = 0;
  po[0] = 0;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* it = items[i];
    Py_ssize_t L;
    if (PyTuple_CheckExact(it)) L = PyTuple_GET_SIZE(it);
    else if (PyList_CheckExact(it)) L = PyList_GET_SIZE(it);
    else {
      L = PySequence_Size(it);
      if (L < 0) {
        PyErr_Clear();
        Py_INCREF(Py_None);
        ret = Py_None;
        goto done;
      }
    }
    total += L;
    if (total > 0x7fffffffLL) {
      PyErr_SetString(PyExc_OverflowError, "corpus has more than 2^31-1 tokens");
      goto done;
    }
    po[i + 1] = (int32_t)total;
  }
  tok = PyByteArray_FromStringAndSize(NULL, (Py_ssize_t)total * (Py_ssize_t)sizeof(int32_t));
  if (!tok) goto done;
  int32_t* pt = (int32_t*)PyByteArray_AS_STRING(tok);
  int ok = 1;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* it = items[i];
    const Py_ssize_t L = po[i + 1] - po[i];
    if (L == 0) ok = 0;
    PyObject* f = PySequence_Fast(it, "input must be a sequence");
    if (!f) {
      PyErr_Clear();
      Py_INCREF(Py_None);
      ret = Py_None;
      goto done;
    }
    if (PySequence_Fast_GET_SIZE(f) != L) {  /* changed under us */
      Py_DECREF(f);
      Py_INCREF(Py_None);
      ret = Py_None;
      goto done;
    }
    PyObject** e = PySequence_Fast_ITEMS(f);
    int32_t* dst = pt + po[i];
    for (Py_ssize_t j = 0; j < L; ++j) {
      long long t;
#if PY_VERSION_HEX >= 0x030C0000
      if (PyLong_CheckExact(e[j]) && PyUnstable_Long_IsCompact((PyLongObject*)e[j]))
        t = (long long)PyUnstable_Long_CompactValue((PyLongObject*)e[j]);
      else
#endif
        t = PyLong_AsLongLong(e[j]);
      if (t == -1 && PyErr_Occurred()) {
        PyErr_Clear();
        Py_DECREF(f);
        Py_INCREF(Py_None);
        ret = Py_None;
        goto done;
      }
      if (t < 0 || t >= V) ok = 0;
      dst[j] = (int32_t)t;
    }
    Py_DECREF(f);
  }
  ret = Py_BuildValue("(OOi)", tok, off, ok);
done:
  Py_XDECREF(tok);
  Py_XDECREF(off);
  Py_DECREF(seq);
  return ret;
}

static PyMethodDef methods[] = {
    {"flatten", flatten, METH_VARARGS, "Flatten a corpus to int32 tokens + offsets, range-checked."},
    {"fill", fill, METH_VARARGS, "Build Candidate lists for a chunk of decoded inputs."},
    {"reserve", reserve, METH_VARARGS, "Cache the int objects of token ids [0, V)."},
    {"fill_packed", fill_packed, METH_VARARGS, "Build Candidate lists from a packed (gathered) shard."},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_vsmat", NULL, -1, methods};

PyMODINIT_FUNC PyInit__vsmat(void) { return PyModule_Create(&moddef); }
