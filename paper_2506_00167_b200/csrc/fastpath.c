/*
 * fastpath.c — CPython entry for the drop-in single-slot build_codebook.
 *
 * The reference call (engine.py:97-116) spends microseconds per slot in
 * interpreter dispatch alone: four Generator.standard_normal calls
 * (sac.py:351-353), array conversions and tuple building.  This module does
 * the same work in one C call on top of the C ABI (include/cyrus_b200.h):
 *
 *   - branch noise: random_standard_normal_fill on each branch generator's
 *     bitgen_t — the exact function Generator.standard_normal(E) runs
 *     (numpy/random/_generator.pyx), so the draws and the generator state
 *     advance are bit-identical to the reference's (tests/test_host.py);
 *   - one cyr_codebook_host call (K2 + K3 on the GPU, GIL released);
 *   - the Codebook.columns tuple of tuples of Python ints.
 *
 * Like numpy's own C-API users this bypasses the Generator's Python-level
 * lock: one build_codebook per Streams object at a time (the reference's
 * Streams are not thread-safe either).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <time.h>

#include "cyrus_b200.h"

typedef struct bitgen {
  void* state;
  uint64_t (*next_uint64)(void* st);
  uint32_t (*next_uint32)(void* st);
  double (*next_double)(void* st);
  uint64_t (*next_raw)(void* st);
} bitgen_t;

/* numpy/random/lib/libnpyrandom.a */
void random_standard_normal_fill(bitgen_t* bitgen_state, Py_ssize_t cnt, double* out);

#define MAX_USERS 32
#define MAX_BRANCHES 16

static int64_t now_ns(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

/* draw(bitgen_addresses, E) -> list of cap lists: test hook for the noise */
static PyObject* fp_draw(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 2 || !PyTuple_Check(args[0])) {
    PyErr_SetString(PyExc_TypeError, "draw(bitgens: tuple, E: int)");
    return NULL;
  }
  const Py_ssize_t cap = PyTuple_GET_SIZE(args[0]);
  const long E = PyLong_AsLong(args[1]);
  if (E < 1 || E > MAX_USERS || cap > MAX_BRANCHES) {
    PyErr_SetString(PyExc_ValueError, "bad sizes");
    return NULL;
  }
  PyObject* out = PyList_New(cap);
  for (Py_ssize_t j = 0; j < cap; ++j) {
    double eps[MAX_USERS];
    bitgen_t* bg = (bitgen_t*)PyLong_AsVoidPtr(PyTuple_GET_ITEM(args[0], j));
    random_standard_normal_fill(bg, E, eps);
    PyObject* row = PyList_New(E);
    for (long e = 0; e < E; ++e) PyList_SET_ITEM(row, e, PyFloat_FromDouble(eps[e]));
    PyList_SET_ITEM(out, j, row);
  }
  return out;
}

/*
 * codebook(policy, alloc, bitgens, N, L, E) -> (status, columns, gen_ns, device_ns)
 *   policy:  cyr_policy* address (int)
 *   alloc:   tuple/sequence of E ints (ScheduleVector.alloc)
 *   bitgens: tuple of cap bitgen_t* addresses (stochastic) or None
 *            (deterministic actor mean, sac.py:349-350)
 * status != 0 leaves columns None; the caller raises the reference's error.
 */
static PyObject* fp_codebook(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 6) {
    PyErr_SetString(PyExc_TypeError, "codebook(policy, alloc, bitgens, N, L, E)");
    return NULL;
  }
  const int64_t t0 = now_ns();
  void* policy = PyLong_AsVoidPtr(args[0]);
  const long N = PyLong_AsLong(args[3]);
  const long L = PyLong_AsLong(args[4]);
  const long E = PyLong_AsLong(args[5]);
  if (PyErr_Occurred()) return NULL;
  if (E < 1 || E > MAX_USERS || L <= 0 || N <= 0) {
    PyErr_SetString(PyExc_ValueError, "bad cell geometry");
    return NULL;
  }
  const long cap = N / L;
  PyObject* seq = PySequence_Fast(args[1], "alloc must be a sequence");
  if (!seq) return NULL;
  if (PySequence_Fast_GET_SIZE(seq) != E) {
    Py_DECREF(seq);
    PyErr_SetString(PyExc_ValueError, "input must be (input_dim, batch)");
    return NULL;
  }
  int32_t alloc[MAX_USERS];
  for (long e = 0; e < E; ++e) {
    const long v = PyLong_AsLong(PySequence_Fast_GET_ITEM(seq, e));
    alloc[e] = (int32_t)v;
  }
  Py_DECREF(seq);
  if (PyErr_Occurred()) return NULL;

  double eps[MAX_BRANCHES * MAX_USERS];
  const double* eps_ptr = NULL;
  if (args[2] != Py_None) {
    if (!PyTuple_Check(args[2]) || PyTuple_GET_SIZE(args[2]) != cap || cap > MAX_BRANCHES) {
      PyErr_SetString(PyExc_ValueError, "need one branch generator per codebook column");
      return NULL;
    }
    for (long j = 0; j < cap; ++j) {
      bitgen_t* bg = (bitgen_t*)PyLong_AsVoidPtr(PyTuple_GET_ITEM(args[2], j));
      if (!bg) return NULL;
      random_standard_normal_fill(bg, E, eps + j * E);
    }
    eps_ptr = eps;
  }

  int32_t book[(MAX_BRANCHES + 1) * MAX_USERS];
  int64_t dev_ns = 0;
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = cyr_codebook_host((cyr_policy*)policy, alloc, eps_ptr, 1, (int32_t)N, (int32_t)L, book,
                             &dev_ns);
  Py_END_ALLOW_THREADS
  const int64_t gen_ns = now_ns() - t0;
  if (status != CYR_OK) return Py_BuildValue("(iOLL)", status, Py_None, (long long)gen_ns, 0LL);

  PyObject* cols = PyTuple_New(cap + 1);
  for (long j = 0; j <= cap; ++j) {
    PyObject* row = PyTuple_New(E);
    for (long e = 0; e < E; ++e) PyTuple_SET_ITEM(row, e, PyLong_FromLong(book[j * E + e]));
    PyTuple_SET_ITEM(cols, j, row);
  }
  PyObject* res = Py_BuildValue("(iNLL)", status, cols, (long long)gen_ns, (long long)dev_ns);
  return res;
}

/*
 * codebook2(policy, alloc, branch, gens, addrs, N, L, E, weights, biases, arrays)
 *     -> (status, columns, gen_ns, device_ns)
 * The drop-in call with its per-call Python bookkeeping moved here:
 *   branch: streams.branch (dict j -> Generator) or None (deterministic);
 *           gens / addrs: the cached generators of j = 1..cap and their
 *           bitgen_t addresses — each branch[j] must still BE gens[j-1]
 *           (status -101 otherwise: the caller refreshes its cache);
 *   weights, biases: agent.actor's lists; arrays: the host arrays registered
 *           with cyr_policy_watch in flatten order (W0, b0, W1, ...) or None —
 *           every list item must still BE the registered array (status -100
 *           otherwise: an array was replaced, the caller re-registers).
 * In-place content changes are caught by the C library itself
 * (cyr_policy_watch), overlapped with the device work.
 */
#define FP_STALE_ARRAYS (-100)
#define FP_STALE_GENS (-101)

static PyObject* g_branch_keys[MAX_BRANCHES + 1];

static PyObject* fp_codebook2(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 11) {
    PyErr_SetString(PyExc_TypeError,
                    "codebook2(policy, alloc, branch, gens, addrs, N, L, E, weights, biases, arrays)");
    return NULL;
  }
  const int64_t t0 = now_ns();
  void* policy = PyLong_AsVoidPtr(args[0]);
  const long N = PyLong_AsLong(args[5]);
  const long L = PyLong_AsLong(args[6]);
  const long E = PyLong_AsLong(args[7]);
  if (PyErr_Occurred()) return NULL;
  if (E < 1 || E > MAX_USERS || L <= 0 || N <= 0) {
    PyErr_SetString(PyExc_ValueError, "bad cell geometry");
    return NULL;
  }
  const long cap = N / L;
  if (cap > MAX_BRANCHES) {
    PyErr_SetString(PyExc_ValueError, "too many branches");
    return NULL;
  }
  /* registered weight arrays still the actor's */
  PyObject* arrays = args[10];
  if (arrays != Py_None) {
    PyObject* w = args[8];
    PyObject* b = args[9];
    if (!PyList_Check(w) || !PyList_Check(b) || !PyTuple_Check(arrays)) {
      PyErr_SetString(PyExc_TypeError, "weights/biases must be lists, arrays a tuple");
      return NULL;
    }
    const Py_ssize_t nl = PyList_GET_SIZE(w);
    int same = PyList_GET_SIZE(b) == nl && PyTuple_GET_SIZE(arrays) == 2 * nl;
    for (Py_ssize_t l = 0; same && l < nl; ++l)
      same = PyList_GET_ITEM(w, l) == PyTuple_GET_ITEM(arrays, 2 * l) &&
             PyList_GET_ITEM(b, l) == PyTuple_GET_ITEM(arrays, 2 * l + 1);
    if (!same) return Py_BuildValue("(iOLL)", FP_STALE_ARRAYS, Py_None, 0LL, 0LL);
  }
  PyObject* seq = PySequence_Fast(args[1], "alloc must be a sequence");
  if (!seq) return NULL;
  if (PySequence_Fast_GET_SIZE(seq) != E) {
    Py_DECREF(seq);
    PyErr_SetString(PyExc_ValueError, "input must be (input_dim, batch)");
    return NULL;
  }
  int32_t alloc[MAX_USERS];
  for (long e = 0; e < E; ++e) alloc[e] = (int32_t)PyLong_AsLong(PySequence_Fast_GET_ITEM(seq, e));
  Py_DECREF(seq);
  if (PyErr_Occurred()) return NULL;

  double eps[MAX_BRANCHES * MAX_USERS];
  const double* eps_ptr = NULL;
  PyObject* branch = args[2];
  if (branch != Py_None) {
    PyObject* gens = args[3];
    PyObject* addrs = args[4];
    if (!PyDict_Check(branch) || !PyTuple_Check(gens) || !PyTuple_Check(addrs) ||
        PyTuple_GET_SIZE(gens) != cap || PyTuple_GET_SIZE(addrs) != cap)
      return Py_BuildValue("(iOLL)", FP_STALE_GENS, Py_None, 0LL, 0LL);
    for (long j = 1; j <= cap; ++j) {
      if (!g_branch_keys[j]) g_branch_keys[j] = PyLong_FromLong(j);
      if (PyDict_GetItemWithError(branch, g_branch_keys[j]) != PyTuple_GET_ITEM(gens, j - 1)) {
        if (PyErr_Occurred()) return NULL;
        return Py_BuildValue("(iOLL)", FP_STALE_GENS, Py_None, 0LL, 0LL);
      }
    }
    for (long j = 0; j < cap; ++j) {
      bitgen_t* bg = (bitgen_t*)PyLong_AsVoidPtr(PyTuple_GET_ITEM(addrs, j));
      if (!bg) return NULL;
      random_standard_normal_fill(bg, E, eps + j * E);
    }
    eps_ptr = eps;
  }

  int32_t book[(MAX_BRANCHES + 1) * MAX_USERS];
  int64_t dev_ns = 0;
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = cyr_codebook_host((cyr_policy*)policy, alloc, eps_ptr, 1, (int32_t)N, (int32_t)L, book,
                             &dev_ns);
  Py_END_ALLOW_THREADS
  const int64_t gen_ns = now_ns() - t0;
  if (status != CYR_OK) return Py_BuildValue("(iOLL)", status, Py_None, (long long)gen_ns, 0LL);
  PyObject* cols = PyTuple_New(cap + 1);
  for (long j = 0; j <= cap; ++j) {
    PyObject* row = PyTuple_New(E);
    for (long e = 0; e < E; ++e) PyTuple_SET_ITEM(row, e, PyLong_FromLong(book[j * E + e]));
    PyTuple_SET_ITEM(cols, j, row);
  }
  return Py_BuildValue("(iNLL)", status, cols, (long long)gen_ns, (long long)dev_ns);
}

static PyMethodDef methods[] = {
    {"codebook2", (PyCFunction)(void (*)(void))fp_codebook2, METH_FASTCALL,
     "codebook2(policy, alloc, branch, gens, addrs, N, L, E, weights, biases, arrays) -> "
     "(status, columns, gen_ns, device_ns); status -100 / -101: stale arrays / generators"},
    {"codebook", (PyCFunction)(void (*)(void))fp_codebook, METH_FASTCALL,
     "codebook(policy, alloc, bitgens, N, L, E) -> (status, columns, gen_ns, device_ns)"},
    {"draw", (PyCFunction)(void (*)(void))fp_draw, METH_FASTCALL,
     "draw(bitgens, E) -> branch noise rows (test hook)"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_fastpath",
                                    "single-slot build_codebook fast path", -1, methods};

PyMODINIT_FUNC PyInit__fastpath(void) { return PyModule_Create(&module); }
