// Reference batch -> CSR, natively (include/chebm2l_batch.h).
//
// The reference hands apply_level its batch as Python objects (m2l.py:279-305,
// built by engine.py:113-119):
//
//     batch = [(target_row, [(source_row, (t0, t1, t2)), ...]), ...]
//
// A Python loop over that structure costs ~380 ns per pair (20 s for the 52 M
// pairs of BASELINE config 2).  This walks the same objects in C: one pass on
// the calling thread counts the pairs, then worker threads fill the CSR arrays
// over disjoint target ranges.  The caller holds the GIL for the whole call
// (the library is loaded with ctypes.PyDLL), so no Python code can run and
// mutate or free the objects; the workers only read immutable tuples and
// compact ints through field accessors that touch no interpreter state.  Any
// object outside the fast shapes (non-tuple pairs, big ints, numpy scalars)
// makes the call return CFM_BATCH_FALLBACK and the Python shim converts that
// batch itself, so behaviour never depends on this path.
#include <Python.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/chebm2l_batch.h"

namespace {

inline bool seq_items(PyObject* o, PyObject*** items, Py_ssize_t* n) {
  if (PyTuple_Check(o)) {
    *items = &PyTuple_GET_ITEM(o, 0);
    *n = PyTuple_GET_SIZE(o);
    return true;
  }
  if (PyList_Check(o)) {
    *items = reinterpret_cast<PyListObject*>(o)->ob_item;
    *n = PyList_GET_SIZE(o);
    return true;
  }
  return false;
}

inline bool small_int(PyObject* o, int64_t* v) {
  if (!PyLong_CheckExact(o)) return false;
  const PyLongObject* l = reinterpret_cast<const PyLongObject*>(o);
  if (!_PyLong_IsCompact(l)) return false;
  *v = int64_t(_PyLong_CompactValue(l));
  return true;
}

// Fill the pairs of targets [b, e): returns false on an unsupported object.
bool fill_range(PyObject** targets, Py_ssize_t b, Py_ssize_t e, const int64_t* off, int64_t* tgt, int64_t* src,
                int8_t* t) {
  for (Py_ssize_t i = b; i < e; ++i) {
    PyObject** pair;
    Py_ssize_t np;
    if (!seq_items(targets[i], &pair, &np) || np != 2) return false;
    if (!small_int(pair[0], &tgt[i])) return false;
    PyObject** far;
    Py_ssize_t nf;
    if (!seq_items(pair[1], &far, &nf)) return false;
    if (off[i + 1] - off[i] != nf) return false;
    int64_t q = off[i];
    for (Py_ssize_t k = 0; k < nf; ++k, ++q) {
      PyObject** st;
      Py_ssize_t ns;
      if (!seq_items(far[k], &st, &ns) || ns != 2) return false;
      if (!small_int(st[0], &src[q])) return false;
      PyObject** tv;
      Py_ssize_t nt;
      if (!seq_items(st[1], &tv, &nt) || nt != 3) return false;
      for (int a = 0; a < 3; ++a) {
        int64_t c;
        if (!small_int(tv[a], &c)) return false;
        // far outside [-3, 3]: clipped to int8; the native side reports it as a
        // missing operator (PrecomputeIncompleteError), as the Python path does
        t[3 * q + a] = int8_t(std::min<int64_t>(127, std::max<int64_t>(-128, c)));
      }
    }
  }
  return true;
}

}  // namespace

extern "C" {

int cfm_batch_count(void* batch_obj, int64_t* n_targets, int64_t* n_pairs, int64_t* offsets_or_null) {
  PyObject* batch = static_cast<PyObject*>(batch_obj);
  PyObject** items;
  Py_ssize_t n;
  if (!batch || !seq_items(batch, &items, &n)) return CFM_BATCH_FALLBACK;
  int64_t total = 0;
  if (offsets_or_null) offsets_or_null[0] = 0;
  for (Py_ssize_t i = 0; i < n; ++i) {
    PyObject** pair;
    Py_ssize_t np;
    if (!seq_items(items[i], &pair, &np) || np != 2) return CFM_BATCH_FALLBACK;
    PyObject** far;
    Py_ssize_t nf;
    if (!seq_items(pair[1], &far, &nf)) return CFM_BATCH_FALLBACK;
    total += nf;
    if (offsets_or_null) offsets_or_null[i + 1] = total;
  }
  if (n_targets) *n_targets = n;
  if (n_pairs) *n_pairs = total;
  return CFM_BATCH_OK;
}

int cfm_batch_fill(void* batch_obj, const int64_t* off, int64_t* tgt, int64_t* src, int8_t* t, int n_threads) {
  PyObject* batch = static_cast<PyObject*>(batch_obj);
  PyObject** items;
  Py_ssize_t n;
  if (!batch || !seq_items(batch, &items, &n)) return CFM_BATCH_FALLBACK;
  if (n == 0) return CFM_BATCH_OK;
  const int64_t P = off[n];
  int nt = n_threads > 0 ? n_threads : int(std::max(1u, std::thread::hardware_concurrency()));
  nt = int(std::min<int64_t>(nt, std::max<int64_t>(1, P / 200000)));  // ~200 k pairs per worker at least
  if (nt <= 1) return fill_range(items, 0, n, off, tgt, src, t) ? CFM_BATCH_OK : CFM_BATCH_FALLBACK;
  // split targets so every worker gets about P / nt pairs
  std::vector<Py_ssize_t> cut(nt + 1, n);
  cut[0] = 0;
  for (int w = 1; w < nt; ++w)
    cut[w] = Py_ssize_t(std::lower_bound(off, off + n + 1, P * w / nt) - off);
  for (int w = 1; w <= nt; ++w) cut[w] = std::max(cut[w], cut[w - 1]);
  std::atomic<bool> ok{true};
  std::vector<std::thread> pool;
  for (int w = 0; w < nt; ++w)
    pool.emplace_back([&, w] {
      if (!fill_range(items, cut[w], cut[w + 1], off, tgt, src, t)) ok = false;
    });
  for (auto& th : pool) th.join();
  return ok ? CFM_BATCH_OK : CFM_BATCH_FALLBACK;
}

// The reference blocked apply's flush sequence (m2l.py:397-452): pairs are
// appended to their representative's 128-column buffer in batch order, a full
// buffer is flushed at once, and the partial buffers are flushed at the end in
// ascending representative index.  Returns the number of flushes written to
// rep_out/cols_out (capacity cap; -1 if too small or a pair has no rep).
int64_t cfm_flush_sequence(int64_t n_pairs, const int8_t* t, const int16_t* rep_of_code, int n_reps, int block_size,
                           int32_t* rep_out, int32_t* cols_out, int64_t cap) {
  if (block_size <= 0 || n_reps < 0) return -1;
  std::vector<int64_t> cnt(size_t(n_reps), 0);
  int64_t k = 0;
  for (int64_t q = 0; q < n_pairs; ++q) {
    const int code = (t[3 * q] + 3) * 49 + (t[3 * q + 1] + 3) * 7 + (t[3 * q + 2] + 3);
    if (code < 0 || code >= 343) return -1;
    const int r = rep_of_code[code];
    if (r < 0 || r >= n_reps) return -1;
    if (++cnt[r] == block_size) {
      if (k >= cap) return -1;
      rep_out[k] = r;
      cols_out[k++] = block_size;
      cnt[r] = 0;
    }
  }
  for (int r = 0; r < n_reps; ++r)
    if (cnt[r]) {
      if (k >= cap) return -1;
      rep_out[k] = r;
      cols_out[k++] = int32_t(cnt[r]);
    }
  return k;
}

}  // extern "C"
