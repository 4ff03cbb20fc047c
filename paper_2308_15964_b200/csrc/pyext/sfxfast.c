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

#include <stdint.h>

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

/* Process-global task ids (reference task.py:63-69): one atomic counter shared by
 * the single-task fast path and the array submissions (reserve). */
static uint64_t g_next_tid = 1;

/* reserve_tids(n) -> first of n consecutive task ids */
static PyObject* reserve_tids(PyObject* self, PyObject* arg) {
  (void)self;
  const long long n = PyLong_AsLongLong(arg);
  if (n < 0 || PyErr_Occurred()) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "n must be >= 0");
    return NULL;
  }
  return PyLong_FromUnsignedLongLong(__atomic_fetch_add(&g_next_tid, (uint64_t)n, __ATOMIC_RELAXED));
}

static PyObject* g_spec_type = NULL; /* access.AccessSpec */
static PyObject* g_op_type = NULL;   /* ops.Op */
static PyObject *s_mode, *s_obj, *s_view, *s_code, *s_fparam, *s_iparam;

/* bind(AccessSpec, Op): the two classes the fast path accepts */
static PyObject* bind_types(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 2) {
    PyErr_SetString(PyExc_TypeError, "bind_types(AccessSpec, Op)");
    return NULL;
  }
  Py_XDECREF(g_spec_type);
  Py_XDECREF(g_op_type);
  g_spec_type = args[0];
  g_op_type = args[1];
  Py_INCREF(g_spec_type);
  Py_INCREF(g_op_type);
  Py_RETURN_NONE;
}

/* task(rt, gid, hid_by_id, tids, accesses, op, priority) -> tid, or 0 when the
 * fast path does not apply (an unregistered object, an array view, a foreign
 * access type, more than 64 accesses): the caller then takes the Python path.
 * A duplicate object -> -1 (the caller raises DuplicateAccessError); a negative
 * runtime status is returned as is (< -1). */
static PyObject* task(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
  (void)self;
  if (nargs != 7 || !g_spec_type) {
    PyErr_SetString(PyExc_TypeError, "task takes 7 arguments (after bind_types)");
    return NULL;
  }
  PyObject* hid_by_id = args[2];
  PyObject* tids = args[3];
  PyObject* accesses = args[4];
  PyObject* op = args[5];
  if (!PyDict_Check(hid_by_id) || !PyList_Check(tids) || !PyTuple_Check(accesses) ||
      (PyObject*)Py_TYPE(op) != g_op_type)
    return PyLong_FromLong(0);
  const Py_ssize_t n = PyTuple_GET_SIZE(accesses);
  if (n > 64) return PyLong_FromLong(0);
  sfx_access acc[64];
  for (Py_ssize_t k = 0; k < n; ++k) {
    PyObject* spec = PyTuple_GET_ITEM(accesses, k);
    if ((PyObject*)Py_TYPE(spec) != g_spec_type) return PyLong_FromLong(0);
    PyObject* view = PyObject_GetAttr(spec, s_view);
    if (!view) return NULL;
    const int has_view = view != Py_None;
    Py_DECREF(view);
    if (has_view) return PyLong_FromLong(0);
    PyObject* obj = PyObject_GetAttr(spec, s_obj);
    if (!obj) return NULL;
    PyObject* key = PyLong_FromVoidPtr(obj); /* id(obj) */
    Py_DECREF(obj);
    if (!key) return NULL;
    PyObject* hid = PyDict_GetItemWithError(hid_by_id, key); /* borrowed */
    Py_DECREF(key);
    if (!hid) {
      if (PyErr_Occurred()) return NULL;
      return PyLong_FromLong(0); /* first use: the Python path registers it */
    }
    PyObject* code = PyObject_GetAttr(spec, s_code);
    if (!code) return NULL;
    acc[k].hid = (uint64_t)PyLong_AsUnsignedLongLong(hid);
    acc[k].mode = (uint32_t)PyLong_AsUnsignedLong(code);
    acc[k].reserved = 0;
    Py_DECREF(code);
    for (Py_ssize_t j = 0; j < k; ++j)
      if (acc[j].hid == acc[k].hid) return PyLong_FromLong(-1);
  }
  sfx_task_desc d;
  d.graph = (uint32_t)PyLong_AsUnsignedLong(args[1]);
  d.op = 0;
  d.priority = (int32_t)PyLong_AsLong(args[6]);
  d.device = -1;
  d.flags = 0;
  d.n_access = (uint32_t)n;
  PyObject* opcode = PyObject_GetAttr(op, s_code);
  PyObject* fp = PyObject_GetAttr(op, s_fparam);
  PyObject* ip = PyObject_GetAttr(op, s_iparam);
  int bad = !opcode || !fp || !ip || !PyTuple_Check(fp) || PyTuple_GET_SIZE(fp) != 4 || !PyTuple_Check(ip) ||
            PyTuple_GET_SIZE(ip) != 4;
  if (!bad) {
    d.op = (uint32_t)PyLong_AsUnsignedLong(opcode);
    for (int k = 0; k < 4; ++k) {
      d.fparam[k] = PyFloat_AsDouble(PyTuple_GET_ITEM(fp, k));
      d.iparam[k] = (int64_t)PyLong_AsLongLong(PyTuple_GET_ITEM(ip, k));
    }
  }
  Py_XDECREF(opcode);
  Py_XDECREF(fp);
  Py_XDECREF(ip);
  if (bad) {
    if (!PyErr_Occurred()) PyErr_SetString(PyExc_TypeError, "malformed op");
    return NULL;
  }
  if (PyErr_Occurred()) return NULL;
  sfx_runtime* rt = (sfx_runtime*)PyLong_AsVoidPtr(args[0]);
  d.tid = __atomic_fetch_add(&g_next_tid, 1, __ATOMIC_RELAXED);
  const int rc = sfx_submit(rt, 1, &d, acc);
  if (rc < 0) return PyLong_FromLong(rc < -1 ? rc : -2);
  PyObject* t = PyLong_FromUnsignedLongLong(d.tid);
  if (!t) return NULL;
  if (PyList_Append(tids, t) < 0) {
    Py_DECREF(t);
    return NULL;
  }
  return t;
}

static PyMethodDef methods[] = {
    {"submit1", (PyCFunction)(void (*)(void))submit1, METH_FASTCALL, "submit one task descriptor (see sfx.h)"},
    {"task", (PyCFunction)(void (*)(void))task, METH_FASTCALL, "TaskGraph.task fast path (see graph.py)"},
    {"bind_types", (PyCFunction)(void (*)(void))bind_types, METH_FASTCALL, "register AccessSpec and Op"},
    {"reserve_tids", reserve_tids, METH_O, "reserve n consecutive process-global task ids"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_sfxfast", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__sfxfast(void) {
  s_mode = PyUnicode_InternFromString("mode");
  s_obj = PyUnicode_InternFromString("obj");
  s_view = PyUnicode_InternFromString("view");
  s_code = PyUnicode_InternFromString("code");
  s_fparam = PyUnicode_InternFromString("fparam");
  s_iparam = PyUnicode_InternFromString("iparam");
  return PyModule_Create(&module);
}
