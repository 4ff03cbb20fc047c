/* _sfxfast: CPython fast path for TaskGraph.task's native submit (one task).
 *
 * The ctypes route packs two structs with struct.pack_into and crosses the
 * ctypes call machinery (~2 us of the ~7 us a Python-inserted task costs); this
 * module converts the arguments with the C API and calls sfx_submit directly.
 * Same ABI, same semantics: the Python side falls back to ctypes when the
 * module is missing.  Built by paper_2308_15964_b200/build.py (g++, -fPIC,
 * linked against libsfx.so with rpath $ORIGIN).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include "sfx.h"

/* submit1(rt, gid, tid, op, prio, dev, fparam4, iparam4, hids, modes) -> int status */
static PyObject* submit1(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 10) {
    PyErr_SetString(PyExc_TypeError, "submit1 takes 10 arguments");
    return NULL;
  }
  sfx_runtime* rt = (sfx_runtime*)PyLong_AsVoidPtr(args[0]);
  sfx_task_desc d;
  d.graph = (uint32_t)PyLong_AsUnsignedLong(args[1]);
  d.tid = (uint64_t)PyLong_AsUnsignedLongLong(args[2]);
  d.op = (uint32_t)PyLong_AsUnsignedLong(args[3]);
  d.priority = (int32_t)PyLong_AsLong(args[4]);
  d.device = (int32_t)PyLong_AsLong(args[5]);
  d.flags = 0;
  PyObject* fp = args[6];
  PyObject* ip = args[7];
  if (!PyTuple_Check(fp) || PyTuple_GET_SIZE(fp) != 4 || !PyTuple_Check(ip) || PyTuple_GET_SIZE(ip) != 4) {
    PyErr_SetString(PyExc_TypeError, "fparam/iparam must be 4-tuples");
    return NULL;
  }
  for (int k = 0; k < 4; ++k) {
    d.fparam[k] = PyFloat_AsDouble(PyTuple_GET_ITEM(fp, k));
    d.iparam[k] = (int64_t)PyLong_AsLongLong(PyTuple_GET_ITEM(ip, k));
  }
  PyObject* hids = args[8];
  PyObject* modes = args[9];
  if (!PyList_Check(hids) || !PyList_Check(modes) || PyList_GET_SIZE(hids) != PyList_GET_SIZE(modes) ||
      PyList_GET_SIZE(hids) > 64) {
    PyErr_SetString(PyExc_TypeError, "hids/modes must be lists of equal length (<= 64)");
    return NULL;
  }
  const Py_ssize_t n = PyList_GET_SIZE(hids);
  sfx_access acc[64];
  for (Py_ssize_t k = 0; k < n; ++k) {
    acc[k].hid = (uint64_t)PyLong_AsUnsignedLongLong(PyList_GET_ITEM(hids, k));
    acc[k].mode = (uint32_t)PyLong_AsUnsignedLong(PyList_GET_ITEM(modes, k));
    acc[k].reserved = 0;
  }
  d.n_access = (uint32_t)n;
  if (PyErr_Occurred()) return NULL;
  int rc;
  Py_BEGIN_ALLOW_THREADS
  rc = sfx_submit(rt, 1, &d, acc);
  Py_END_ALLOW_THREADS
  return PyLong_FromLong(rc);
}

static PyMethodDef methods[] = {
    {"submit1", (PyCFunction)(void (*)(void))submit1, METH_FASTCALL, "submit one task descriptor (see sfx.h)"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_sfxfast", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__sfxfast(void) { return PyModule_Create(&module); }
