// CPython fast path for the per-call entry points of the reference API
// (allreduce / reduce_scatter / allgather / the fused aggregate call / poll).
//
// The ctypes binding converts every argument through Python objects on each
// call (~5 us for cm_allreduce's 11 arguments); the paper's point is exactly
// this per-call host cost, so the façade calls these thin wrappers instead:
// integers in, the cm status and the CollectiveStats fields out. Errors are
// reported by status; the façade maps them to the reference exception classes
// (and reads cm_last_error) through the ctypes binding, off the fast path.
//
// The module does not link libcm.so: bind() receives the entry points of the
// library instance the ctypes binding loaded, so a CM_LIB override (e.g. the
// checked build) stays one library.
#include <Python.h>

#include "cm.h"

namespace {

decltype(&cm_allreduce) f_allreduce = nullptr;
decltype(&cm_reduce_scatter) f_reduce_scatter = nullptr;
decltype(&cm_allgather) f_allgather = nullptr;
decltype(&cm_fused_allreduce_agreed) f_fused = nullptr;
decltype(&cm_comm_poll) f_poll = nullptr;
decltype(&cm_comm_sync) f_sync = nullptr;

bool bound() {
  if (f_allreduce) return true;
  PyErr_SetString(PyExc_RuntimeError, "_cmfast.bind() was not called");
  return false;
}

// bind(allreduce, reduce_scatter, allgather, fused, poll, sync): addresses
PyObject* py_bind(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 6) {
    PyErr_SetString(PyExc_TypeError, "bind takes 6 function addresses");
    return nullptr;
  }
  void* a[6];
  for (int i = 0; i < 6; ++i) {
    a[i] = PyLong_AsVoidPtr(args[i]);
    if (PyErr_Occurred()) return nullptr;
  }
  f_allreduce = reinterpret_cast<decltype(f_allreduce)>(a[0]);
  f_reduce_scatter = reinterpret_cast<decltype(f_reduce_scatter)>(a[1]);
  f_allgather = reinterpret_cast<decltype(f_allgather)>(a[2]);
  f_fused = reinterpret_cast<decltype(f_fused)>(a[3]);
  f_poll = reinterpret_cast<decltype(f_poll)>(a[4]);
  f_sync = reinterpret_cast<decltype(f_sync)>(a[5]);
  Py_RETURN_NONE;
}

PyObject* stats_tuple(int status, const cm_stats_t& s) {
  return Py_BuildValue("(iLLL)", status, (long long)s.rounds, (long long)s.messages_per_rank,
                       (long long)s.bytes_sent_per_rank);
}

// allreduce(comm, send, recv, count, dtype, op, algo, switch_bytes, average, stream)
PyObject* py_allreduce(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 10) {
    PyErr_SetString(PyExc_TypeError, "allreduce takes 10 integer arguments");
    return nullptr;
  }
  unsigned long long comm = PyLong_AsUnsignedLongLong(args[0]);
  unsigned long long send = PyLong_AsUnsignedLongLong(args[1]);
  unsigned long long recv = PyLong_AsUnsignedLongLong(args[2]);
  long long count = PyLong_AsLongLong(args[3]);
  int dtype = (int)PyLong_AsLong(args[4]);
  int op = (int)PyLong_AsLong(args[5]);
  int algo = (int)PyLong_AsLong(args[6]);
  long long sw = PyLong_AsLongLong(args[7]);
  int avg = (int)PyLong_AsLong(args[8]);
  unsigned long long stream = PyLong_AsUnsignedLongLong(args[9]);
  if (PyErr_Occurred() || !bound()) return nullptr;
  cm_stats_t st{0, 0, 0};
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = f_allreduce(reinterpret_cast<cm_comm_t*>(comm), reinterpret_cast<const void*>(send),
                        reinterpret_cast<void*>(recv), count, dtype, op, algo, sw, avg,
                        reinterpret_cast<void*>(stream), &st);
  Py_END_ALLOW_THREADS
  return stats_tuple(status, st);
}

// reduce_scatter / allgather(comm, send, recv, count, dtype, op_or_layout..., stream)
PyObject* py_reduce_scatter(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 8) {
    PyErr_SetString(PyExc_TypeError, "reduce_scatter takes 8 integer arguments");
    return nullptr;
  }
  unsigned long long comm = PyLong_AsUnsignedLongLong(args[0]);
  unsigned long long send = PyLong_AsUnsignedLongLong(args[1]);
  unsigned long long recv = PyLong_AsUnsignedLongLong(args[2]);
  long long count = PyLong_AsLongLong(args[3]);
  int dtype = (int)PyLong_AsLong(args[4]);
  int op = (int)PyLong_AsLong(args[5]);
  int layout = (int)PyLong_AsLong(args[6]);
  unsigned long long stream = PyLong_AsUnsignedLongLong(args[7]);
  if (PyErr_Occurred() || !bound()) return nullptr;
  cm_stats_t st{0, 0, 0};
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = f_reduce_scatter(reinterpret_cast<cm_comm_t*>(comm), reinterpret_cast<const void*>(send),
                             reinterpret_cast<void*>(recv), count, dtype, op, layout,
                             reinterpret_cast<void*>(stream), &st);
  Py_END_ALLOW_THREADS
  return stats_tuple(status, st);
}

PyObject* py_allgather(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 7) {
    PyErr_SetString(PyExc_TypeError, "allgather takes 7 integer arguments");
    return nullptr;
  }
  unsigned long long comm = PyLong_AsUnsignedLongLong(args[0]);
  unsigned long long send = PyLong_AsUnsignedLongLong(args[1]);
  unsigned long long recv = PyLong_AsUnsignedLongLong(args[2]);
  long long count = PyLong_AsLongLong(args[3]);
  int dtype = (int)PyLong_AsLong(args[4]);
  int layout = (int)PyLong_AsLong(args[5]);
  unsigned long long stream = PyLong_AsUnsignedLongLong(args[6]);
  if (PyErr_Occurred() || !bound()) return nullptr;
  cm_stats_t st{0, 0, 0};
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = f_allgather(reinterpret_cast<cm_comm_t*>(comm), reinterpret_cast<const void*>(send),
                        reinterpret_cast<void*>(recv), count, dtype, layout, reinterpret_cast<void*>(stream), &st);
  Py_END_ALLOW_THREADS
  return stats_tuple(status, st);
}

// fused(comm, n, sends*, counts*, dtype, recv, algo, threshold, switch, average,
//       agree*, n_agree, reg_ids*, stream, stats*) -> (status, agreed, n_calls)
// (pointer arguments are addresses of arrays the façade keeps per plan)
PyObject* py_fused(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 15) {
    PyErr_SetString(PyExc_TypeError, "fused takes 15 integer arguments");
    return nullptr;
  }
  unsigned long long comm = PyLong_AsUnsignedLongLong(args[0]);
  int n = (int)PyLong_AsLong(args[1]);
  unsigned long long sends = PyLong_AsUnsignedLongLong(args[2]);
  unsigned long long counts = PyLong_AsUnsignedLongLong(args[3]);
  int dtype = (int)PyLong_AsLong(args[4]);
  unsigned long long recv = PyLong_AsUnsignedLongLong(args[5]);
  int algo = (int)PyLong_AsLong(args[6]);
  long long threshold = PyLong_AsLongLong(args[7]);
  long long sw = PyLong_AsLongLong(args[8]);
  int avg = (int)PyLong_AsLong(args[9]);
  unsigned long long agree = PyLong_AsUnsignedLongLong(args[10]);
  int n_agree = (int)PyLong_AsLong(args[11]);
  unsigned long long reg = PyLong_AsUnsignedLongLong(args[12]);
  unsigned long long stream = PyLong_AsUnsignedLongLong(args[13]);
  unsigned long long stats = PyLong_AsUnsignedLongLong(args[14]);
  if (PyErr_Occurred() || !bound()) return nullptr;
  int agreed = 1, n_calls = 0, status;
  Py_BEGIN_ALLOW_THREADS
  status = f_fused(
      reinterpret_cast<cm_comm_t*>(comm), n, reinterpret_cast<const void* const*>(sends),
      reinterpret_cast<const int64_t*>(counts), dtype, reinterpret_cast<void*>(recv), algo, threshold, sw, avg,
      reinterpret_cast<const int64_t*>(agree), n_agree, &agreed, reinterpret_cast<const int64_t*>(reg),
      reinterpret_cast<void*>(stream), reinterpret_cast<cm_stats_t*>(stats), &n_calls);
  Py_END_ALLOW_THREADS
  return Py_BuildValue("(iii)", status, agreed, n_calls);
}

PyObject* py_poll(PyObject*, PyObject* arg) {
  unsigned long long comm = PyLong_AsUnsignedLongLong(arg);
  if (PyErr_Occurred() || !bound()) return nullptr;
  return PyLong_FromLong(f_poll(reinterpret_cast<cm_comm_t*>(comm)));
}

PyObject* py_sync(PyObject*, PyObject* const* args, Py_ssize_t nargs) {
  if (nargs != 2) {
    PyErr_SetString(PyExc_TypeError, "sync takes (comm, stream)");
    return nullptr;
  }
  unsigned long long comm = PyLong_AsUnsignedLongLong(args[0]);
  unsigned long long stream = PyLong_AsUnsignedLongLong(args[1]);
  if (PyErr_Occurred() || !bound()) return nullptr;
  int status;
  Py_BEGIN_ALLOW_THREADS
  status = f_sync(reinterpret_cast<cm_comm_t*>(comm), reinterpret_cast<void*>(stream));
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(status);
}

PyMethodDef methods[] = {
    {"bind", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(py_bind)), METH_FASTCALL,
     "bind(allreduce, reduce_scatter, allgather, fused, poll, sync) entry-point addresses"},
    {"allreduce", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(py_allreduce)), METH_FASTCALL,
     "cm_allreduce -> (status, rounds, messages, bytes)"},
    {"reduce_scatter", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(py_reduce_scatter)),
     METH_FASTCALL, "cm_reduce_scatter -> (status, rounds, messages, bytes)"},
    {"allgather", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(py_allgather)), METH_FASTCALL,
     "cm_allgather -> (status, rounds, messages, bytes)"},
    {"fused", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(py_fused)), METH_FASTCALL,
     "cm_fused_allreduce_agreed -> (status, agreed, n_calls)"},
    {"poll", py_poll, METH_O, "cm_comm_poll -> status"},
    {"sync", reinterpret_cast<PyCFunction>(reinterpret_cast<void (*)(void)>(py_sync)), METH_FASTCALL,
     "cm_comm_sync -> status"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef module = {PyModuleDef_HEAD_INIT, "_cmfast", "CPython fast path over libcm.so", -1, methods,
                      nullptr, nullptr, nullptr, nullptr};

}  // namespace

PyMODINIT_FUNC PyInit__cmfast(void) { return PyModule_Create(&module); }
