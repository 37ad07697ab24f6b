// _pdb_host: native result materialisation.
//
// The reference returns the determinant as a CoeffTensor whose coefficients
// are Python ints (crt.py:122-130).  After the GPU CRT the coefficients exist
// as little-endian u32 magnitude limbs + sign bytes; turning 10^6-10^7 of them
// into Python ints one `int.from_bytes` call at a time costs ~0.3-0.7 us each
// in the interpreter.  This module does the same conversion in one C loop
// (PyLong from the limb bytes, negated where the sign byte is set), writing
// the coefficient tuple directly, zeros as the shared small int 0.
//
//   ints_from_limbs(limbs: bytes-like [count][width] u32, index: bytes-like int64[count],
//                   neg: bytes-like uint8[count], n: int, width: int) -> tuple[int] of length n
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <cstdint>
#include <cstring>

// On other interpreters (or with PDB_NO_DIRECT_LONG) every coefficient takes the
// portable path below, which uses the public API only.
// CPython 3.12/3.13 store an int as 30-bit digits behind a tag word
// (digit count << 3 | sign: 0 positive, 2 negative).  Building the object
// directly from the limb bit stream skips _PyLong_FromByteArray's byte loop
// and, for negative values, the second allocation of PyNumber_Negative.
#if PY_VERSION_HEX >= 0x030C0000 && PY_VERSION_HEX < 0x030E0000 && PYLONG_BITS_IN_DIGIT == 30 && \
    !defined(PDB_NO_DIRECT_LONG)
#define PDB_DIRECT_LONG 1
static PyObject* long_from_limbs(const unsigned char* row, Py_ssize_t width, bool negative) {
  digit buf[80];   // up to 74 limbs = 2368 bits
  Py_ssize_t nd = 0;
  uint64_t acc = 0;
  int bits = 0;
  for (Py_ssize_t w = 0; w < width; ++w) {
    uint32_t limb;
    std::memcpy(&limb, row + 4 * w, 4);
    acc |= (uint64_t)limb << bits;
    bits += 32;
    while (bits >= PyLong_SHIFT) {
      buf[nd++] = (digit)(acc & PyLong_MASK);
      acc >>= PyLong_SHIFT;
      bits -= PyLong_SHIFT;
    }
  }
  if (bits > 0) buf[nd++] = (digit)acc;
  while (nd > 0 && buf[nd - 1] == 0) --nd;
  if (nd <= 2) {   // fits in 60 bits: the public constructor (keeps small ints canonical)
    long long v = nd == 0 ? 0 : (long long)buf[0] | (nd == 2 ? (long long)buf[1] << PyLong_SHIFT : 0);
    return PyLong_FromLongLong(negative ? -v : v);
  }
  PyLongObject* op = _PyLong_New(nd);
  if (!op) return nullptr;
  std::memcpy(op->long_value.ob_digit, buf, (size_t)nd * sizeof(digit));
  if (negative) op->long_value.lv_tag = ((uintptr_t)nd << _PyLong_NON_SIZE_BITS) | 2;
  return (PyObject*)op;
}
#endif

// Portable path (public API only, any CPython): int.from_bytes(row, "little").
static PyObject* g_from_bytes = nullptr;   // bound method int.from_bytes

static PyObject* portable_int(const unsigned char* row, Py_ssize_t width) {
  if (width <= 2) {
    uint64_t mag = 0;
    std::memcpy(&mag, row, (size_t)width * 4);
    return PyLong_FromUnsignedLongLong(mag);
  }
  if (!g_from_bytes) {
    g_from_bytes = PyObject_GetAttrString((PyObject*)&PyLong_Type, "from_bytes");
    if (!g_from_bytes) return nullptr;
  }
  return PyObject_CallFunction(g_from_bytes, "y#s", (const char*)row, width * 4, "little");
}

// One coefficient: |value| as `width` little-endian u32 limbs, then the sign.
static PyObject* make_int(const unsigned char* row, Py_ssize_t width, bool negative, bool portable) {
#ifdef PDB_DIRECT_LONG
  if (!portable && width <= 74) return long_from_limbs(row, width, negative);
#else
  (void)portable;
#endif
  PyObject* v = portable_int(row, width);
  if (v && negative) {
    PyObject* m = PyNumber_Negative(v);
    Py_DECREF(v);
    v = m;
  }
  return v;
}

static PyObject* build(PyObject* args, bool portable) {
  Py_buffer limbs, index, neg;
  Py_ssize_t n, width;
  if (!PyArg_ParseTuple(args, "y*y*y*nn", &limbs, &index, &neg, &n, &width)) return nullptr;
  PyObject* out = nullptr;
  const Py_ssize_t count = index.len / (Py_ssize_t)sizeof(int64_t);
  const unsigned char* lb = static_cast<const unsigned char*>(limbs.buf);
  const int64_t* ix = static_cast<const int64_t*>(index.buf);
  const uint8_t* ng = static_cast<const uint8_t*>(neg.buf);
  bool sorted = true;
  PyObject* zero = nullptr;
  if (width < 1 || n < 0 || limbs.len != count * width * 4 || neg.len != count) {
    PyErr_SetString(PyExc_ValueError, "ints_from_limbs: inconsistent buffer sizes");
    goto done;
  }
  for (Py_ssize_t j = 0; j < count; ++j) {
    if (ix[j] < 0 || ix[j] >= n) {
      PyErr_SetString(PyExc_IndexError, "ints_from_limbs: index out of range");
      goto done;
    }
    if (j && ix[j] <= ix[j - 1]) sorted = false;
  }
  // the result is the coefficient tuple itself (CoeffTensor.coeffs), built in one pass
  out = PyTuple_New(n);
  if (!out) goto done;
  zero = PyLong_FromLong(0);
  if (sorted) {
    Py_ssize_t j = 0;
    for (Py_ssize_t i = 0; i < n; ++i) {
      PyObject* v;
      if (j < count && ix[j] == i) {
        v = make_int(lb + (size_t)j * (size_t)width * 4, width, ng[j] != 0, portable);
        ++j;
        if (!v) { Py_CLEAR(out); goto done; }
      } else {
        Py_INCREF(zero);
        v = zero;
      }
      PyTuple_SET_ITEM(out, i, v);
    }
  } else {   // any order (duplicates: the last wins), before the tuple escapes
    for (Py_ssize_t i = 0; i < n; ++i) {
      Py_INCREF(zero);
      PyTuple_SET_ITEM(out, i, zero);
    }
    for (Py_ssize_t j = 0; j < count; ++j) {
      PyObject* v = make_int(lb + (size_t)j * (size_t)width * 4, width, ng[j] != 0, portable);
      if (!v) { Py_CLEAR(out); goto done; }
      PyObject* old = PyTuple_GET_ITEM(out, ix[j]);
      PyTuple_SET_ITEM(out, ix[j], v);
      Py_DECREF(old);
    }
  }
done:
  Py_XDECREF(zero);
  PyBuffer_Release(&limbs);
  PyBuffer_Release(&index);
  PyBuffer_Release(&neg);
  return out;
}

static PyObject* ints_from_limbs(PyObject*, PyObject* args) { return build(args, false); }
static PyObject* ints_from_limbs_portable(PyObject*, PyObject* args) { return build(args, true); }

static PyObject* direct_path(PyObject*, PyObject*) {
#ifdef PDB_DIRECT_LONG
  Py_RETURN_TRUE;
#else
  Py_RETURN_FALSE;
#endif
}

static PyMethodDef methods[] = {
    {"ints_from_limbs", ints_from_limbs, METH_VARARGS,
     "ints_from_limbs(limbs, index, neg, n, width) -> tuple of n Python ints"},
    {"ints_from_limbs_portable", ints_from_limbs_portable, METH_VARARGS,
     "the same through the public C API only (int.from_bytes): the path on other CPython ABIs"},
    {"direct_path", direct_path, METH_NOARGS, "True if this build writes PyLong digits directly"},
    {nullptr, nullptr, 0, nullptr}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pdb_host", "native result materialisation", -1, methods};

PyMODINIT_FUNC PyInit__pdb_host(void) { return PyModule_Create(&module); }
