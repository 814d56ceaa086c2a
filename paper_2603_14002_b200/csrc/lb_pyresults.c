/* lb_pyresults.c -- CPython binding that turns an lb_results_view (include/lightbeam_b200.h)
 * into the decode results the Python API returns:
 *
 *     assemble(view_address) -> [None | (best_text, best_score, [(text, score), ...])]
 *
 * one entry per trial, None for trials whose status is not 0.  The strings are decoded straight
 * from the library's text blob (no intermediate bytes object, no split), so a config-2 batch
 * (256 trials, ~15k n-best texts, ~5 MB of text) costs one pass over the blob.  Same objects as
 * `DeviceBatch.results()` built them in Python (decoder.py:433-460 result shape).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include "lightbeam_b200.h"

static PyObject* assemble(PyObject* self, PyObject* arg) {
  (void)self;
  const lb_results_view* v = (const lb_results_view*)PyLong_AsVoidPtr(arg);
  if (v == NULL) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "null results view");
    return NULL;
  }
  const int n = v->n_trials;
  PyObject* out = PyList_New(n);
  if (!out) return NULL;
  /* ~15k tuples per config-2 batch: keep the cyclic GC from running generations over them
   * while they are built (none of these objects can form a cycle) */
  const int gc_was_enabled = PyGC_Disable();
  int64_t j = 0;
  for (int i = 0; i < n; ++i) {
    if (v->status[i] != 0) {
      Py_INCREF(Py_None);
      PyList_SET_ITEM(out, i, Py_None);
      continue;
    }
    const int c = v->nbest_count[i];
    if (j + c > v->total_nbest) {
      Py_DECREF(out);
      PyErr_SetString(PyExc_RuntimeError, "results view is inconsistent");
      if (gc_was_enabled) PyGC_Enable();
      return NULL;
    }
    PyObject* best = PyUnicode_DecodeUTF8(v->blob + v->best_text_off[i], v->best_text_len[i], "strict");
    PyObject* bsc = PyFloat_FromDouble(v->best_score[i]);
    PyObject* nb = PyList_New(c);
    if (!best || !bsc || !nb) goto fail_item;
    for (int q = 0; q < c; ++q, ++j) {
      PyObject* tx = PyUnicode_DecodeUTF8(v->blob + v->nbest_text_off[j], v->nbest_text_len[j], "strict");
      PyObject* sc = PyFloat_FromDouble(v->nbest_score[j]);
      PyObject* pr = (tx && sc) ? PyTuple_Pack(2, tx, sc) : NULL;
      Py_XDECREF(tx);
      Py_XDECREF(sc);
      if (!pr) goto fail_item;
      /* a (str, float) pair can never be part of a reference cycle: keep it out of the cyclic
       * GC's young generation, which otherwise re-traverses ~15k of them per batch */
      PyObject_GC_UnTrack(pr);
      PyList_SET_ITEM(nb, q, pr);
    }
    {
      PyObject* item = PyTuple_Pack(3, best, bsc, nb);
      Py_DECREF(best);
      Py_DECREF(bsc);
      Py_DECREF(nb);
      if (!item) {
        Py_DECREF(out);
        if (gc_was_enabled) PyGC_Enable();
        return NULL;
      }
      PyList_SET_ITEM(out, i, item);
    }
    continue;
  fail_item:
    Py_XDECREF(best);
    Py_XDECREF(bsc);
    Py_XDECREF(nb);
    Py_DECREF(out);
    if (gc_was_enabled) PyGC_Enable();
    return NULL;
  }
  if (gc_was_enabled) PyGC_Enable();
  return out;
}

static PyMethodDef methods[] = {
    {"assemble", assemble, METH_O, "lb_results_view address -> per-trial results"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_lb_results", NULL, -1, methods};

PyMODINIT_FUNC PyInit__lb_results(void) { return PyModule_Create(&module); }
