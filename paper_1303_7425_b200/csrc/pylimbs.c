/* pylimbs.c -- host-side marshaling of exact integer coefficients.
 *
 * The GPU returns integer coefficients as 1-3 little-endian u64 limbs of two's
 * complement per term; the reference's Polynomial holds Python ints
 * (core.py:231-241).  Building 10^5-10^8 Python ints one by one in Python
 * costs ~200 ns each; this module builds them in C (PyLong_FromLongLong when
 * the value fits 64 bits, else _PyLong_FromByteArray on the limb bytes).
 * Marshaling only: no arithmetic on coefficients happens here.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>
#include <string.h>

static PyObject* limbs_to_list(PyObject* self, PyObject* args) {
  Py_buffer buf;
  Py_ssize_t n, nl;
  if (!PyArg_ParseTuple(args, "y*nn", &buf, &n, &nl)) return NULL;
  if (nl < 1 || nl > 8 || buf.len < n * nl * 8) {
    PyBuffer_Release(&buf);
    PyErr_SetString(PyExc_ValueError, "buffer too small for n terms of nl limbs");
    return NULL;
  }
  const uint64_t* w = (const uint64_t*)buf.buf;
  PyObject* out = PyList_New(n);
  if (!out) {
    PyBuffer_Release(&buf);
    return NULL;
  }
  for (Py_ssize_t i = 0; i < n; ++i) {
    const uint64_t* t = w + i * nl;
    const uint64_t sign = (uint64_t)((int64_t)t[0] >> 63);
    int small = 1;
    for (Py_ssize_t k = 1; k < nl; ++k)
      if (t[k] != sign) {
        small = 0;
        break;
      }
    PyObject* v = small ? PyLong_FromLongLong((long long)t[0])
                        : _PyLong_FromByteArray((const unsigned char*)t, (size_t)(8 * nl), 1, 1);
    if (!v) {
      Py_DECREF(out);
      PyBuffer_Release(&buf);
      return NULL;
    }
    PyList_SET_ITEM(out, i, v);
  }
  PyBuffer_Release(&buf);
  return out;
}

static PyMethodDef methods[] = {
    {"limbs_to_list", limbs_to_list, METH_VARARGS,
     "limbs_to_list(buffer, n, nl) -> list of n Python ints from nl little-endian u64 limbs each"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pylimbs", NULL, -1, methods};

PyMODINIT_FUNC PyInit__pylimbs(void) { return PyModule_Create(&module); }
