/*
 * chebm2l_batch — the reference's Python batch -> CSR arrays, in C
 * (libcfm_batch.so; loaded with ctypes.PyDLL so the GIL is held throughout).
 *
 *   reference                                          replaced by
 *   -----------------------------------------------    --------------------------
 *   apply_level(level, batch, ...)  m2l.py:279-305     cfm_batch_count +
 *     batch = [(row, [(src, t), ...]), ...]              cfm_batch_fill, then
 *     built by FmmPlan._level_data  engine.py:113-119    cfm_apply_level_csr
 *
 * `batch_obj` is the PyObject* of the batch (a list or tuple of 2-sequences
 * (target_row, far_list); far_list items are (source_row, (t0, t1, t2))),
 * passed as a plain pointer; no other Python type appears here.
 * Returns CFM_BATCH_OK, or CFM_BATCH_FALLBACK when an object is outside the
 * fast shapes (the caller then converts in Python; nothing was raised).
 */
#ifndef CHEBM2L_BATCH_H
#define CHEBM2L_BATCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CFM_BATCH_OK 0
#define CFM_BATCH_FALLBACK 1

/* Number of targets and pairs; offsets_or_null (n_targets + 1 int64, may be
 * NULL on a sizing call) receives the CSR offsets. */
int cfm_batch_count(void* batch_obj, int64_t* n_targets, int64_t* n_pairs, int64_t* offsets_or_null);

/* Fill target rows tgt[n], source rows src[P] and transfer vectors t[3P]
 * (int8, clipped) given the offsets of cfm_batch_count; n_threads <= 0 = all
 * hardware threads. */
int cfm_batch_fill(void* batch_obj, const int64_t* off, int64_t* tgt, int64_t* src, int8_t* t, int n_threads);

/* Block statistics of the reference's blocked apply (m2l.py:397-452, the
 * `products` / `flushes` of block_stats): the flush sequence of a batch's
 * pairs (t[3P] in batch order) for buffers of block_size columns.
 * rep_of_code[343] maps a t-code to its representative index (-1 = none).
 * Writes (rep index, columns) per flush in the reference's order and returns
 * the count, or -1 (capacity cap too small, or a pair without a rep).
 * No Python objects involved. */
int64_t cfm_flush_sequence(int64_t n_pairs, const int8_t* t, const int16_t* rep_of_code, int n_reps,
                           int block_size, int32_t* rep_out, int32_t* cols_out, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif
