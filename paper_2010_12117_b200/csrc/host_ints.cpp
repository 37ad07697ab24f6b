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

// ---- format_terms: the reference's canonical polynomial text at 10^5-10^7 terms ----
//
// format_terms(terms: dict[tuple[int, ...], int], variables: tuple[str, ...], threads: int) -> str
// byte-identical to parsing.py:197-225 (format_polynomial): terms sorted by
// (total degree, exponent tuple) descending; a term prints its variables with
// exponent 1 as `x`, > 1 as `x^e` (others omitted), joined by `*`, prefixed by
// `|c|*` unless |c| = 1 (a constant prints |c|); the first term carries `-` for
// a negative coefficient, later ones are joined as ` + t` / ` - t`; no terms
// prints `0`.  Keys must be tuples of exact ints of one arity and values exact
// ints (the caller normalises anything else first, tensor.py:25-32); zero
// coefficients are skipped.  The sort and the text run in C++ (the decimal
// digits of big coefficients in `threads` threads on CPython 3.12/3.13).
#include <algorithm>
#include <deque>
#include <string>
#include <thread>
#include <vector>

namespace {

struct FmtTerm {
  const int64_t* e;   // exponents (arity k)
  int64_t deg;
  PyObject* c;        // borrowed coefficient
  bool neg, one;      // c < 0, |c| == 1 (read with the GIL, before the threads start)
  const std::string* dec;   // |c| in decimal when made with the GIL (huge or portable), else null
};

// |v| in decimal, appended to out.  Direct path: 30-bit digits -> base 10^9 by
// schoolbook division (no Python API: safe in worker threads).
static bool append_abs_decimal(std::string& out, PyObject* v) {
#ifdef PDB_DIRECT_LONG
  const PyLongObject* op = reinterpret_cast<const PyLongObject*>(v);
  const uintptr_t tag = op->long_value.lv_tag;
  Py_ssize_t nd = (Py_ssize_t)(tag >> _PyLong_NON_SIZE_BITS);
  const digit* d = op->long_value.ob_digit;
  if (nd == 0) { out.push_back('0'); return true; }
  if (nd <= 2) {
    unsigned long long m = d[0] | (nd == 2 ? (unsigned long long)d[1] << PyLong_SHIFT : 0ull);
    char buf[24];
    int n = 0;
    do { buf[n++] = (char)('0' + m % 10); m /= 10; } while (m);
    while (n) out.push_back(buf[--n]);
    return true;
  }
  if (nd > 80) return false;
  uint32_t w[80];                        // little-endian base 2^30
  for (Py_ssize_t i = 0; i < nd; ++i) w[i] = d[i];
  uint32_t chunks[100];                  // base 10^9, little-endian
  int nc = 0;
  Py_ssize_t top = nd;
  while (top > 0) {
    uint64_t rem = 0;
    for (Py_ssize_t i = top - 1; i >= 0; --i) {
      const uint64_t cur = (rem << PyLong_SHIFT) | w[i];
      const uint64_t q = cur / 1000000000ull;
      w[i] = (uint32_t)q;
      rem = cur - q * 1000000000ull;
    }
    chunks[nc++] = (uint32_t)rem;
    while (top > 0 && w[top - 1] == 0) --top;
  }
  char buf[16];
  int n = 0;
  uint32_t x = chunks[nc - 1];
  do { buf[n++] = (char)('0' + x % 10); x /= 10; } while (x);
  while (n) out.push_back(buf[--n]);
  for (int i = nc - 2; i >= 0; --i) {
    x = chunks[i];
    char nine[9];
    for (int j = 8; j >= 0; --j) { nine[j] = (char)('0' + x % 10); x /= 10; }
    out.append(nine, 9);
  }
  return true;
#else
  (void)out; (void)v;
  return false;
#endif
}

struct FmtCtx {
  std::vector<FmtTerm>* terms;
  int k;
  const std::vector<std::string>* names;
};

static void format_range(const FmtCtx& cx, size_t lo, size_t hi, std::string& out) {
  const std::vector<FmtTerm>& T = *cx.terms;
  for (size_t i = lo; i < hi; ++i) {
    const FmtTerm& t = T[i];
    const bool neg = t.neg;
    if (i == 0) {
      if (neg) out.push_back('-');
    } else {
      out.append(neg ? " - " : " + ");
    }
    bool body = false;
    for (int a = 0; a < cx.k; ++a) if (t.e[a] >= 1) { body = true; break; }
    const bool one = body && t.one;
    if (!one) {
      if (t.dec) out.append(*t.dec);
      else append_abs_decimal(out, t.c);
      if (body) out.push_back('*');
    }
    bool first = true;
    for (int a = 0; a < cx.k; ++a) {
      const int64_t e = t.e[a];
      if (e < 1) continue;
      if (!first) out.push_back('*');
      first = false;
      out.append((*cx.names)[a]);
      if (e > 1) {
        out.push_back('^');
        out.append(std::to_string((long long)e));
      }
    }
  }
}

}  // namespace

// One coefficient into the term list (GIL held): its sign, |c| == 1, and for
// huge or portable-build magnitudes the decimal digits made now.
static bool fmt_add(std::vector<FmtTerm>& T, std::deque<std::string>& decs, PyObject* val) {
#ifdef PDB_DIRECT_LONG
  const uintptr_t tag = reinterpret_cast<const PyLongObject*>(val)->long_value.lv_tag;
  const bool neg = (tag & 3) == 2;
  const bool one = (tag >> _PyLong_NON_SIZE_BITS) == 1 && reinterpret_cast<const PyLongObject*>(val)->long_value.ob_digit[0] == 1;
  const bool huge = (tag >> _PyLong_NON_SIZE_BITS) > 80;
#else
  PyObject* zero_obj = PyLong_FromLong(0);
  const int n0 = PyObject_RichCompareBool(val, zero_obj, Py_LT);
  Py_DECREF(zero_obj);
  if (n0 < 0) return false;
  const bool neg = n0 == 1;
  PyObject* a1 = PyNumber_Absolute(val);
  if (!a1) return false;
  PyObject* one_obj = PyLong_FromLong(1);
  const bool one = PyObject_RichCompareBool(a1, one_obj, Py_EQ) == 1;
  Py_DECREF(one_obj);
  Py_DECREF(a1);
  const bool huge = true;   // portable build: every magnitude through the public API
#endif
  const std::string* dec = nullptr;
  if (huge) {
    PyObject* a = PyNumber_Absolute(val);
    PyObject* str = a ? PyObject_Str(a) : nullptr;
    Py_XDECREF(a);
    if (!str) return false;
    Py_ssize_t sn = 0;
    const char* u = PyUnicode_AsUTF8AndSize(str, &sn);
    decs.emplace_back(u, (size_t)sn);
    Py_DECREF(str);
    dec = &decs.back();
  }
  T.push_back(FmtTerm{nullptr, 0, val, neg, one, dec});
  return true;
}

static bool fmt_names(PyObject* variables, std::vector<std::string>& names) {
  const int k = (int)PyTuple_GET_SIZE(variables);
  names.assign((size_t)k, std::string());
  for (int a = 0; a < k; ++a) {
    Py_ssize_t n = 0;
    const char* u = PyUnicode_AsUTF8AndSize(PyTuple_GET_ITEM(variables, a), &n);
    if (!u) return false;
    names[(size_t)a].assign(u, (size_t)n);
  }
  return true;
}

// Sort (graded lexicographic, highest first) and print the collected terms.
static PyObject* fmt_finish(std::vector<FmtTerm>& T, std::vector<int64_t>& exps, int k,
                            const std::vector<std::string>& names, int threads) {
  const size_t stride = (size_t)(k > 0 ? k : 1);
  for (size_t i = 0; i < T.size(); ++i) {
    T[i].e = exps.data() + i * stride;
    int64_t d = 0;
    for (int a = 0; a < k; ++a) d += T[i].e[a];
    T[i].deg = d;
  }
  if (T.empty()) return PyUnicode_FromString("0");
  auto later = [k](const FmtTerm& x, const FmtTerm& y) {
    if (x.deg != y.deg) return x.deg > y.deg;
    for (int a = 0; a < k; ++a)
      if (x.e[a] != y.e[a]) return x.e[a] > y.e[a];
    return false;
  };
  const int nthreads = std::max(1, std::min(threads, 64));
  Py_BEGIN_ALLOW_THREADS
  {
    // chunks sorted in parallel, then merged pairwise (each round in parallel)
    const size_t n = T.size();
    const int ns = n < 100000 ? 1 : nthreads;
    std::vector<size_t> cut((size_t)ns + 1);
    for (int j = 0; j <= ns; ++j) cut[(size_t)j] = n * (size_t)j / (size_t)ns;
    std::vector<std::thread> pool;
    for (int j = 0; j < ns; ++j)
      pool.emplace_back([&, j]() { std::sort(T.begin() + cut[(size_t)j], T.begin() + cut[(size_t)j + 1], later); });
    for (auto& th : pool) th.join();
    for (size_t width = 1; width < (size_t)ns; width *= 2) {
      std::vector<std::thread> mp;
      for (size_t j = 0; j + width < (size_t)ns; j += 2 * width) {
        const size_t lo = cut[j], mid = cut[j + width], hi = cut[std::min(j + 2 * width, (size_t)ns)];
        mp.emplace_back([&, lo, mid, hi]() { std::inplace_merge(T.begin() + lo, T.begin() + mid, T.begin() + hi, later); });
      }
      for (auto& th : mp) th.join();
    }
  }
  Py_END_ALLOW_THREADS
  const int nt = T.size() < 20000 ? 1 : nthreads;
  FmtCtx cx{&T, k, &names};
  std::vector<std::string> parts((size_t)nt);
  // the coefficient objects are immutable and kept alive by the caller's
  // container for the whole call: worker threads read their digits without the GIL
  Py_BEGIN_ALLOW_THREADS
  std::vector<std::thread> pool;
  for (int j = 0; j < nt; ++j) {
    const size_t lo = T.size() * (size_t)j / (size_t)nt, hi = T.size() * (size_t)(j + 1) / (size_t)nt;
    auto job = [&cx, &parts, j, lo, hi]() { format_range(cx, lo, hi, parts[(size_t)j]); };
    if (j + 1 < nt) pool.emplace_back(job);
    else job();
  }
  for (auto& th : pool) th.join();
  Py_END_ALLOW_THREADS
  size_t total = 0;
  for (auto& s : parts) total += s.size();
  bool ascii = true;
  for (auto& nm : names)
    for (unsigned char ch : nm) ascii = ascii && ch < 128;
  if (ascii) {   // digits, signs and ASCII names: one copy into the str object
    PyObject* out = PyUnicode_New((Py_ssize_t)total, 127);
    if (!out) return nullptr;
    char* dst = reinterpret_cast<char*>(PyUnicode_1BYTE_DATA(out));
    for (auto& s : parts) {
      std::memcpy(dst, s.data(), s.size());
      dst += s.size();
      std::string().swap(s);
    }
    return out;
  }
  std::string all;
  all.reserve(total);
  for (auto& s : parts) { all.append(s); std::string().swap(s); }
  return PyUnicode_DecodeUTF8(all.data(), (Py_ssize_t)all.size(), "strict");
}

static PyObject* format_terms(PyObject*, PyObject* args) {
  PyObject *terms, *variables;
  int threads = 1;
  if (!PyArg_ParseTuple(args, "O!O!i", &PyDict_Type, &terms, &PyTuple_Type, &variables, &threads)) return nullptr;
  std::vector<std::string> names;
  if (!fmt_names(variables, names)) return nullptr;
  const int k = (int)names.size();
  const Py_ssize_t count = PyDict_GET_SIZE(terms);
  std::vector<int64_t> exps;
  exps.reserve((size_t)count * (size_t)(k > 0 ? k : 1));
  std::vector<FmtTerm> T;
  T.reserve((size_t)count);
  std::deque<std::string> decs;   // stable addresses
  Py_ssize_t pos = 0;
  PyObject *key, *val;
  while (PyDict_Next(terms, &pos, &key, &val)) {
    if (!PyTuple_CheckExact(key) || PyTuple_GET_SIZE(key) != k || !PyLong_CheckExact(val)) {
      PyErr_SetString(PyExc_TypeError, "format_terms: keys must be k-tuples of ints and values ints");
      return nullptr;
    }
    const int zero = PyObject_Not(val);
    if (zero < 0) return nullptr;
    if (zero) continue;
    for (int a = 0; a < k; ++a) {
      PyObject* x = PyTuple_GET_ITEM(key, a);
      if (!PyLong_CheckExact(x)) {
        PyErr_SetString(PyExc_TypeError, "format_terms: exponents must be ints");
        return nullptr;
      }
      const long long e = PyLong_AsLongLong(x);
      if (e == -1 && PyErr_Occurred()) return nullptr;
      exps.push_back((int64_t)e);
    }
    if (k == 0) exps.push_back(0);
    if (!fmt_add(T, decs, val)) return nullptr;
  }
  return fmt_finish(T, exps, k, names, threads);
}

// format_dense(coeffs: tuple of ints (row-major over shape), shape: tuple, variables, threads) -> str:
// the same text for a dense coefficient tensor (CoeffTensor) without building its terms() dict.
static PyObject* format_dense(PyObject*, PyObject* args) {
  PyObject *coeffs, *shape, *variables;
  int threads = 1;
  if (!PyArg_ParseTuple(args, "O!O!O!i", &PyTuple_Type, &coeffs, &PyTuple_Type, &shape, &PyTuple_Type, &variables,
                        &threads))
    return nullptr;
  std::vector<std::string> names;
  if (!fmt_names(variables, names)) return nullptr;
  const int k = (int)names.size();
  if (PyTuple_GET_SIZE(shape) != k) {
    PyErr_SetString(PyExc_ValueError, "format_dense: shape and variables differ in length");
    return nullptr;
  }
  std::vector<int64_t> dims((size_t)k);
  Py_ssize_t n = 1;
  for (int a = 0; a < k; ++a) {
    dims[(size_t)a] = PyLong_AsLongLong(PyTuple_GET_ITEM(shape, a));
    if (dims[(size_t)a] < 1) {
      if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "format_dense: bad shape");
      return nullptr;
    }
    n *= (Py_ssize_t)dims[(size_t)a];
  }
  if (PyTuple_GET_SIZE(coeffs) != n) {
    PyErr_SetString(PyExc_ValueError, "format_dense: coefficient count does not fill the shape");
    return nullptr;
  }
  std::vector<int64_t> exps;
  std::vector<FmtTerm> T;
  std::deque<std::string> decs;
  std::vector<int64_t> idx((size_t)(k > 0 ? k : 1), 0);
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject* val = PyTuple_GET_ITEM(coeffs, i);
    if (!PyLong_CheckExact(val)) {
      PyErr_SetString(PyExc_TypeError, "format_dense: coefficients must be ints");
      return nullptr;
    }
    const int zero = PyObject_Not(val);
    if (zero < 0) return nullptr;
    if (!zero) {
      for (int a = 0; a < k; ++a) exps.push_back(idx[(size_t)a]);
      if (k == 0) exps.push_back(0);
      if (!fmt_add(T, decs, val)) return nullptr;
    }
    for (int a = k - 1; a >= 0; --a) {   // row-major successor of the multi-index
      if (++idx[(size_t)a] < dims[(size_t)a]) break;
      idx[(size_t)a] = 0;
    }
  }
  return fmt_finish(T, exps, k, names, threads);
}

// ints_from_digits(digits: [count][D] u32 30-bit digits, ndig: uint8[count], index: int64[count] (ascending),
//                  neg: uint8[count], n, D) -> tuple of n ints (the device already re-cut the limbs,
//                  pdb_limbs_to_digits30: one allocation + one copy per int; CPython 3.12/3.13 only)
static PyObject* ints_from_digits(PyObject*, PyObject* args) {
#ifdef PDB_DIRECT_LONG
  Py_buffer digits, ndig, index, neg;
  Py_ssize_t n, D;
  if (!PyArg_ParseTuple(args, "y*y*y*y*nn", &digits, &ndig, &index, &neg, &n, &D)) return nullptr;
  PyObject* out = nullptr;
  PyObject* zero = nullptr;
  const Py_ssize_t count = index.len / (Py_ssize_t)sizeof(int64_t);
  const uint32_t* dg = static_cast<const uint32_t*>(digits.buf);
  const uint8_t* nd = static_cast<const uint8_t*>(ndig.buf);
  const int64_t* ix = static_cast<const int64_t*>(index.buf);
  const uint8_t* ng = static_cast<const uint8_t*>(neg.buf);
  if (D < 1 || n < 0 || digits.len != count * D * 4 || ndig.len != count || neg.len != count) {
    PyErr_SetString(PyExc_ValueError, "ints_from_digits: inconsistent buffer sizes");
    goto done;
  }
  for (Py_ssize_t j = 0; j < count; ++j) {
    if (ix[j] < 0 || ix[j] >= n || (j && ix[j] <= ix[j - 1]) || nd[j] > D) {
      PyErr_SetString(PyExc_IndexError, "ints_from_digits: index out of range or not ascending");
      goto done;
    }
  }
  out = PyTuple_New(n);
  if (!out) goto done;
  zero = PyLong_FromLong(0);
  {
    Py_ssize_t j = 0;
    for (Py_ssize_t i = 0; i < n; ++i) {
      PyObject* v;
      if (j < count && ix[j] == i) {
        const Py_ssize_t k = nd[j];
        const uint32_t* row = dg + (size_t)j * (size_t)D;
        const bool negative = ng[j] != 0;
        if (k <= 2) {
          const long long x = k == 0 ? 0 : (long long)row[0] | (k == 2 ? (long long)row[1] << PyLong_SHIFT : 0);
          v = PyLong_FromLongLong(negative ? -x : x);
        } else {
          PyLongObject* op = _PyLong_New(k);
          if (op) {
            std::memcpy(op->long_value.ob_digit, row, (size_t)k * sizeof(digit));
            if (negative) op->long_value.lv_tag = ((uintptr_t)k << _PyLong_NON_SIZE_BITS) | 2;
          }
          v = (PyObject*)op;
        }
        ++j;
        if (!v) { Py_CLEAR(out); goto done; }
      } else {
        Py_INCREF(zero);
        v = zero;
      }
      PyTuple_SET_ITEM(out, i, v);
    }
  }
done:
  Py_XDECREF(zero);
  PyBuffer_Release(&digits);
  PyBuffer_Release(&ndig);
  PyBuffer_Release(&index);
  PyBuffer_Release(&neg);
  return out;
#else
  (void)args;
  PyErr_SetString(PyExc_NotImplementedError, "ints_from_digits needs the direct PyLong layout (CPython 3.12/3.13)");
  return nullptr;
#endif
}

// ints_from_digits_mt(digits, ndig, index, neg, n, D, threads): ints_from_digits
// with the allocation spread over threads.  At 10^6-10^7 coefficients the
// serial builder is bound by the object allocator and the first touch of its
// fresh pages (~100 ns per 449-bit int).  Here each thread builds the int
// objects of a slice of the tuple with the raw (thread-safe) allocator while
// the GIL is released: an int object is its header (refcount 1, &PyLong_Type,
// tag word) and its digits, and CPython frees any object through
// PyObject_Free, which hands addresses outside its own arenas to
// PyMem_RawFree (the path every large object takes).  The caller uses it only
// when no allocation hook is active (tracemalloc, PYTHONMALLOC=debug).  Zeros
// are the shared immortal small int 0 (3.12+), so no refcount is touched.
// (not on free-threaded builds: their object allocator, mimalloc, frees only its own blocks)
#if defined(PDB_DIRECT_LONG) && !defined(Py_REF_DEBUG) && !defined(Py_TRACE_REFS) && !defined(Py_GIL_DISABLED)
#define PDB_MT_LONG 1
static PyObject* raw_long(const uint32_t* row, Py_ssize_t k, bool negative) {
  const size_t bytes = offsetof(PyLongObject, long_value.ob_digit) + (size_t)(k ? k : 1) * sizeof(digit);
  PyLongObject* op = static_cast<PyLongObject*>(PyMem_RawMalloc(bytes));
  if (!op) return nullptr;
  Py_SET_REFCNT((PyObject*)op, 1);
  Py_SET_TYPE((PyObject*)op, &PyLong_Type);
  op->long_value.lv_tag = ((uintptr_t)k << _PyLong_NON_SIZE_BITS) | (negative ? 2u : 0u);
  std::memcpy(op->long_value.ob_digit, row, (size_t)k * sizeof(digit));
  return (PyObject*)op;
}
#endif

static PyObject* ints_from_digits_mt(PyObject*, PyObject* args) {
#ifdef PDB_MT_LONG
  Py_buffer digits, ndig, index, neg;
  Py_ssize_t n, D;
  int threads;
  if (!PyArg_ParseTuple(args, "y*y*y*y*nni", &digits, &ndig, &index, &neg, &n, &D, &threads)) return nullptr;
  PyObject* out = nullptr;
  PyObject* zero = PyLong_FromLong(0);
  const Py_ssize_t count = index.len / (Py_ssize_t)sizeof(int64_t);
  const uint32_t* dg = static_cast<const uint32_t*>(digits.buf);
  const uint8_t* nd = static_cast<const uint8_t*>(ndig.buf);
  const int64_t* ix = static_cast<const int64_t*>(index.buf);
  const uint8_t* ng = static_cast<const uint8_t*>(neg.buf);
  bool failed = false;
  if (D < 1 || n < 0 || digits.len != count * D * 4 || ndig.len != count || neg.len != count) {
    PyErr_SetString(PyExc_ValueError, "ints_from_digits_mt: inconsistent buffer sizes");
    goto done;
  }
  if (!_Py_IsImmortal(zero)) {
    PyErr_SetString(PyExc_RuntimeError, "ints_from_digits_mt: small int 0 is not immortal");
    goto done;
  }
  for (Py_ssize_t j = 0; j < count; ++j) {
    if (ix[j] < 0 || ix[j] >= n || (j && ix[j] <= ix[j - 1]) || nd[j] > D) {
      PyErr_SetString(PyExc_IndexError, "ints_from_digits_mt: index out of range or not ascending");
      goto done;
    }
  }
  out = PyTuple_New(n);
  if (!out) goto done;
  {
    if (threads < 1) threads = 1;
    if (threads > 64) threads = 64;
    PyObject** items = ((PyTupleObject*)out)->ob_item;
    std::vector<char> bad((size_t)threads, 0);
    Py_BEGIN_ALLOW_THREADS
    auto work = [&](int t) {
      const Py_ssize_t lo = n * t / threads, hi = n * (t + 1) / threads;
      Py_ssize_t j = std::lower_bound(ix, ix + count, (int64_t)lo) - ix;
      for (Py_ssize_t i = lo; i < hi; ++i) {
        PyObject* v = zero;
        if (j < count && ix[j] == i) {
          if (nd[j] > 2) {
            v = raw_long(dg + (size_t)j * (size_t)D, nd[j], ng[j] != 0);
            if (!v) { bad[(size_t)t] = 1; v = zero; }
          } else if (nd[j]) {
            v = nullptr;   // <= 60 bits: the public constructor below, with the GIL
          }
          ++j;
        }
        items[i] = v;
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (char b : bad) failed = failed || b;
    Py_END_ALLOW_THREADS
  }
  if (failed) {
    Py_CLEAR(out);
    PyErr_NoMemory();
    goto done;
  }
  for (Py_ssize_t j = 0; j < count; ++j) {   // 1-2 digit values: canonical small ints where they exist
    if (nd[j] == 0 || nd[j] > 2) continue;
    const uint32_t* row = dg + (size_t)j * (size_t)D;
    const long long x = (long long)row[0] | (nd[j] == 2 ? (long long)row[1] << PyLong_SHIFT : 0);
    PyObject* v = PyLong_FromLongLong(ng[j] ? -x : x);
    if (!v) { Py_CLEAR(out); goto done; }
    PyTuple_SET_ITEM(out, ix[j], v);
  }
done:
  Py_XDECREF(zero);
  PyBuffer_Release(&digits);
  PyBuffer_Release(&ndig);
  PyBuffer_Release(&index);
  PyBuffer_Release(&neg);
  return out;
#else
  (void)args;
  PyErr_SetString(PyExc_NotImplementedError, "ints_from_digits_mt needs the direct PyLong layout (CPython 3.12/3.13)");
  return nullptr;
#endif
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
    {"ints_from_digits", ints_from_digits, METH_VARARGS,
     "ints_from_digits(digits, ndig, index, neg, n, D) -> tuple of n ints from device-made 30-bit digit rows"},
    {"ints_from_digits_mt", ints_from_digits_mt, METH_VARARGS,
     "ints_from_digits_mt(digits, ndig, index, neg, n, D, threads): the same, objects built by threads"},
    {"format_dense", format_dense, METH_VARARGS,
     "format_dense(coeffs, shape, variables, threads) -> format_terms of a dense coefficient tensor"},
    {"format_terms", format_terms, METH_VARARGS,
     "format_terms(terms, variables, threads) -> the reference's canonical polynomial text (parsing.py:211-225)"},
    {nullptr, nullptr, 0, nullptr}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_pdb_host", "native result materialisation", -1, methods};

PyMODINIT_FUNC PyInit__pdb_host(void) { return PyModule_Create(&module); }
