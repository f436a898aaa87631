/*
 * chebm2l — B200-native M2L application for the Chebyshev-interpolation
 * black-box FMM (arXiv 1210.7292), C ABI.
 *
 * This is the drop-in boundary for the reference's M2L handler
 * (/root/reference/pkg/src/chebfmm/m2l.py, class M2LHandler :90-536).  The
 * reference is pure Python and has no FFI of its own; these entry points are
 * what a binding of that handler needs (INTEGRATION.md shows the ctypes stub):
 *
 *   reference (m2l.py)                         replaced by
 *   ---------------------------------------    ------------------------------------
 *   M2LHandler.__init__            :93-130     cfm_handler_create
 *   _build_group (dense cache)     :188-194    cfm_set_dense_group
 *   _build_group (low-rank cache)  :197-199    cfm_set_lowrank_group
 *   _build_shared_basis            :216-273    cfm_set_shared_group
 *   precompute level->group/scale  :143-167    cfm_set_level
 *   apply_level                    :279-305    cfm_apply_level_csr / cfm_apply_planned
 *   (_apply_plain/_sym/_shared/_blocked :320-452 are selected by the variant)
 *   octree.build_interaction_lists far part (octree.py:148-178) + symmetry
 *   canonicalize (symmetry.py:63-75)           cfm_classify_count / cfm_classify_fill,
 *                                              cfm_classify_targets_* (a rank's targets)
 *   aca (lowrank.py:65-160) per operator       cfm_aca_batch (compression="aca")
 *   FmmPlan._m2l batches (engine.py:140-157)   cfm_last_csr_plan_info (plan cache of batches)
 *   (multi-GPU halo, no reference counterpart) cfm_gather_rows
 *
 * Conventions (all bit-for-bit those of the reference):
 *   - flat node index m = a1 + a2*l + a3*l^2 (first component fastest), interp.py:134-161;
 *   - transfer vector t = ijk_target - ijk_source, far iff t.t > 3, octree.py:50-65;
 *   - t-code = (t0+3)*49 + (t1+3)*7 + (t2+3) in [0, 343);
 *   - perm id = (f0 | f1<<1 | f2<<2)*6 + rank of axis_order in
 *     [(1,2,3),(1,3,2),(2,1,3),(2,3,1),(3,1,2),(3,2,1)], symmetry.py:63-75;
 *   - operators are row-major, rows = target nodes, cols = source nodes
 *     (kernels.py:125-131); complex scalars are interleaved (re, im) doubles.
 *
 * Error handling: every function returns 0 (CFM_OK) or a CFM_ERR_* code and
 * records a message retrievable with cfm_last_error() (thread-local).  No C++
 * exception crosses the ABI.  The Python shim maps CFM_ERR_VALUE -> ValueError,
 * CFM_ERR_PRECOMPUTE -> PrecomputeIncompleteError (KeyError), CFM_ERR_BUDGET ->
 * BudgetExceededError (RuntimeError), everything else -> RuntimeError.
 *
 * Memory: mpoles/locals pointers may be host or device memory (detected with
 * cudaPointerGetAttributes).  Host buffers are staged through the handler's
 * device scratch (only the rows a batch reads / writes; pageable memory through
 * pinned slots on several host threads); device buffers are used in place.  `stream` is a
 * cudaStream_t (NULL = the CUDA default stream, so work is ordered with the
 * caller's default-stream work).  Calls on one handler are
 * serialized by an internal mutex (the reference may call apply_level from
 * several threads, engine.py:145-155).
 */
#ifndef CHEBM2L_H
#define CHEBM2L_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CFM_OK 0
#define CFM_ERR_VALUE 1
#define CFM_ERR_PRECOMPUTE 2
#define CFM_ERR_BUDGET 3
#define CFM_ERR_CUDA 4
#define CFM_ERR_INTERNAL 5

/* variants, in the reference's VARIANTS order (m2l.py:51) */
#define CFM_NA 0
#define CFM_NASYM 1
#define CFM_NABLK 2
#define CFM_SA 3
#define CFM_SARCMP 4
#define CFM_IA 5
#define CFM_IASYM 6
#define CFM_IABLK 7

#define CFM_N_TCODES 343

typedef struct cfm_handler cfm_handler;

/* Message of the last failing call on this thread ("" if none). */
const char* cfm_last_error(void);

/* ABI version (bumped on any signature change). */
int cfm_abi_version(void);

/* Create a handler bound to CUDA device `device` for one variant, Chebyshev
 * order `order` (n = order^3 nodes) and operator scalar kind
 * (op_complex = 0: float64 operators, 1: complex128).  m2l.py:93-130. */
int cfm_handler_create(int device, int variant, int order, int op_complex, cfm_handler** out);
int cfm_handler_destroy(cfm_handler* h);

/* Every group carries its transfer list (the reference's _Group.transfers,
 * m2l.py:84-87): only those vectors are applicable; any other raises
 * CFM_ERR_PRECOMPUTE like the reference's cache lookups (m2l.py:312-318).
 *
 * Dense operator group (na: one operator per transfer vector; nasym/nablk: one
 * per cone representative).  op_t: n_ops int8 triples; ops: n_ops * n * n
 * scalars (x2 doubles when op_complex).  m2l.py:188-194. */
int cfm_set_dense_group(cfm_handler* h, int key, int n_transfers, const int8_t* transfers,
                        int n_ops, const int8_t* op_t, const double* ops);

/* Low-rank group (ia: per transfer vector; iasym/iablk: per representative).
 * Operator i is left_i (n x r_i, singular values folded) times right_i^H
 * (right_i: n x r_i).  left/right are the row-major blocks concatenated in op
 * order.  lowrank.py:23-44, m2l.py:197-214. */
int cfm_set_lowrank_group(cfm_handler* h, int key, int n_transfers, const int8_t* transfers,
                          int n_ops, const int8_t* op_t, const int32_t* ranks,
                          const double* left, const double* right);

/* Shared-basis group (sa/sarcmp): u (n x r_u), b (n x r_b), and one core per
 * transfer vector: core_rank[i] < 0 -> dense core (r_u x r_b); otherwise a
 * factored core left (r_u x r) and right (r_b x r), core = left @ right^H.
 * core_data concatenates the blocks in core order.  m2l.py:216-273. */
int cfm_set_shared_group(cfm_handler* h, int key, int r_u, int r_b, const double* u,
                         const double* b, int n_cores, const int8_t* core_t,
                         const int32_t* core_rank, const double* core_data);

/* Level -> group key and homogeneous scale (m2l.py:143-167). */
int cfm_set_level(cfm_handler* h, int level, int key, double scale);

/* Apply one level for a batch given in CSR form: target rows tgt[n_targets],
 * pair offsets off[n_targets+1], source rows src[P], transfer vectors t[3P].
 * data_complex: 0 float64 expansions, 1 complex128.  mpoles/locals are
 * n_rows x n (row-major); locals is accumulated in place (+=).
 * pair_count_out (optional, 343 int64): pairs per t-code, for the flop model.
 * m2l.py:279-305. */
int cfm_apply_level_csr(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt,
                        const int64_t* off, const int64_t* src, const int8_t* t,
                        int data_complex, const double* mpoles, int64_t n_rows,
                        double* locals, void* stream, int64_t* pair_count_out);

/* Build and cache the device plan of a level from the sorted occupied cells
 * (ijk int32 triples, lexicographic order = row order, octree.py:124-126): the
 * far lists are classified on the GPU (no host lists).  Then apply it any
 * number of times with cfm_apply_planned. */
int cfm_plan_level_cells(cfm_handler* h, int level, int64_t n_cells, const int32_t* ijk,
                         int data_complex, void* stream, int64_t* pair_count_out);
int cfm_plan_level_csr(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt,
                       const int64_t* off, const int64_t* src, const int8_t* t,
                       int data_complex, int64_t n_rows, int64_t* pair_count_out);
/* As cfm_plan_level_cells, but only for the targets in target_rows (a
 * multi-GPU rank's Morton range of the level).  Optionally returns the sorted
 * source rows those targets read (sources_out must hold n_cells entries): the
 * rows a rank must own or receive in the halo exchange. */
int cfm_plan_level_cells_subset(cfm_handler* h, int level, int64_t n_cells, const int32_t* ijk, int64_t n_targets,
                                const int64_t* target_rows, int data_complex, void* stream, int64_t* pair_count_out,
                                int64_t* n_sources_out, int64_t* sources_out);
int cfm_apply_planned(cfm_handler* h, int level, const double* mpoles, int64_t n_rows,
                      double* locals, void* stream);

/* Apply several planned levels of one M2L step together (the levels are
 * independent, m2l.py:279 per level): dense variants run as ONE kernel launch
 * over all levels' tiles, so small levels overlap the large one.  Arrays are
 * indexed by position; pointers may be host or device memory. */
int cfm_apply_levels(cfm_handler* h, int n_levels, const int* levels, const double* const* mpoles,
                     const int64_t* n_rows, double* const* locals, void* stream);

/* Plan statistics: tiles, entries (GEMM tile products), pairs, entry column
 * slots (entries * 64), distinct targets and distinct sources. */
int cfm_plan_stats(cfm_handler* h, int level, int64_t* n_tiles, int64_t* n_entries,
                   int64_t* n_pairs, int64_t* n_slots, int64_t* n_targets, int64_t* n_sources);

/* Device-output classifier (all pointers device, work on `stream`):
 * offsets_dev gets n_cells+1 int64 CSR offsets (total returned on the host);
 * fill writes per pair the source row (int32) and t-code (int16). */
int cfm_classify_count_device(int device, int level, int64_t n_cells, const int32_t* ijk, int64_t* offsets_dev,
                              int64_t* total_out, void* stream);
int cfm_classify_fill_device(int device, int level, int64_t n_cells, const int32_t* ijk, const int64_t* offsets_dev,
                             int32_t* src_dev, int16_t* code_dev, void* stream);

/* Plan layout chosen for a level: mode 0 = target tiles (per-target register
 * accumulators; dense trees), 1 = pair entries + ordered per-target reduction
 * (sparse trees, chosen when target tiles would be < 60% full; override with
 * CFM_PLAN_MODE=target|pair).  target_fill = pairs / target-tile slots. */
int cfm_plan_info(cfm_handler* h, int level, int* mode, double* target_fill);

/* 1 when a low-rank level (ia / iasym / iablk, real operators, target tiles)
 * runs as two stages: Y = V_t^H x for every (source, transfer of its class) as
 * a dense GEMM, then locals += U_t Y per target tile (m2l.py:425 split at the
 * rank-r intermediate); 0 for the fused single-kernel path.  CFM_LR_TWOSTAGE=0
 * at precompute disables it. */
int cfm_plan_two_stage(cfm_handler* h, int level, int* two_stage);

/* Interaction-list classifier (octree.py:148-178 + symmetry.py:63-75) on the
 * GPU.  Cells: sorted occupied ijk of `level` (int32 triples, host or device).
 * count: per-cell far-pair counts -> offsets (n_cells+1, host int64), returns
 * the total.  fill: per pair, in the reference's order (targets by row, sources
 * by ijk): source row, t (int8 triple), cone representative index into the
 * 16-vector cone (sorted), perm id.  Output arrays are host pointers. */
int cfm_classify_count(int device, int level, int64_t n_cells, const int32_t* ijk,
                       int64_t* offsets_out, int64_t* total_out);
int cfm_classify_fill(int device, int level, int64_t n_cells, const int32_t* ijk,
                      const int64_t* offsets, int32_t* src_out, int8_t* t_out,
                      uint8_t* rep_out, uint8_t* perm_out);

/* The far lists of a subset of a level's cells as targets (a multi-GPU
 * rank's Morton range): sources are all n_cells occupied
 * cells (host ijk), targets are target_rows[n_targets]; offsets_out has
 * n_targets + 1 entries, src_out holds global source rows, t_out t[3P].
 * Same lists and order as octree.py:148-178 for those targets. */
int cfm_classify_targets_count(int device, int level, int64_t n_cells, const int32_t* ijk,
                               int64_t n_targets, const int64_t* target_rows,
                               int64_t* offsets_out, int64_t* total_out);
int cfm_classify_targets_fill(int device, int level, int64_t n_cells, const int32_t* ijk,
                              int64_t n_targets, const int64_t* target_rows,
                              const int64_t* offsets, int32_t* src_out, int8_t* t_out);

/* Partially pivoted ACA (lowrank.py:65-160) of n_ops operators [n_ops][n][n]
 * (device, row-major, complex interleaved when data_complex), one CTA per
 * operator, the reference's pivoting and stopping rule at accuracy eps.
 * u_out / v_out (device, [n_ops][kmax][n]): cross q of operator o in row q
 * (A ~ sum_q u_q v_q^T before conjugation, lowrank.py:152-153).
 * rank_out / flag_out (host, n_ops): crosses, 1 converged / 0 stagnated /
 * 2 more than kmax crosses needed.  m2l.py:206-214, 241-255. */
int cfm_aca_batch(int device, int n, int data_complex, int n_ops, const double* ops, double eps,
                  int kmax, double* u_out, double* v_out, int* rank_out, int* flag_out, void* stream);

/* Multi-GPU halo packing: dst[k, :] = src[rows[k], :] for rows of
 * row_doubles doubles (device pointers; rows int64 on the device). */
int cfm_gather_rows(int device, const double* src, int64_t row_doubles, const int64_t* rows,
                    int64_t n, double* dst, void* stream);

/* Octree construction on the GPU (octree.py:93-127):
 * points n x 3 (host or device), bounding cube (center, half_width), depth
 * >= 2.  Per level: occupied cells in the reference's row order
 * (lexicographic ijk); leaf particle lists as CSR (offsets per leaf, particle
 * indices ascending inside a leaf).  Particles outside the cube ->
 * CFM_ERR_VALUE ("particle outside bounding box"), like the reference. */
typedef struct cfm_tree cfm_tree;
int cfm_tree_build(int device, const double* points, int64_t n, const double* center, double half_width, int depth,
                   cfm_tree** out);
int cfm_tree_level_size(cfm_tree* t, int level, int64_t* n_cells);
int cfm_tree_level_cells(cfm_tree* t, int level, int32_t* ijk_out);
int cfm_tree_leaf_particles(cfm_tree* t, int64_t* offsets_out, int64_t* perm_out);
int cfm_tree_destroy(cfm_tree* t);

/* The FMM stages around M2L on the GPU, on a tree
 * from cfm_tree_build.  shift_mats: 8 octant matrices (parent x child, n x n,
 * octant = 4 cx + 2 cy + cz; engine.py:41-63).  All arrays are device
 * pointers; level arrays are rows x n (x2 doubles when complex), rows in the
 * tree's row order; potentials are in the original particle order.
 *   p2m  engine.py:122-127   m2m engine.py:129-138 (child level -> parent, +=)
 *   l2l  engine.py:159-168 (parent level -> child, +=)
 *   l2p  engine.py:170-175 (+=)   p2p engine.py:177-199 (+=; kernel 0 Laplace
 *   1/(4 pi r), 1 Helmholtz exp(ikr)/(4 pi r); coincident points skipped) */
typedef struct cfm_fmm cfm_fmm;
int cfm_fmm_create(cfm_tree* t, int order, const double* shift_mats, cfm_fmm** out);
int cfm_fmm_destroy(cfm_fmm* f);
int cfm_fmm_p2m(cfm_fmm* f, const double* weights, int data_complex, double* leaf_mpoles, void* stream);
int cfm_fmm_m2m(cfm_fmm* f, int child_level, const double* child, double* parent, int data_complex, void* stream);
int cfm_fmm_l2l(cfm_fmm* f, int parent_level, const double* parent, double* child, int data_complex, void* stream);
int cfm_fmm_l2p(cfm_fmm* f, const double* leaf_locals, int data_complex, double* potentials, void* stream);
int cfm_fmm_p2p(cfm_fmm* f, int kernel, double wavenumber, const double* weights, int weights_complex,
                double* potentials, int out_complex, void* stream);

/* GPU operator assembly (replaces assemble_for_transfer, kernels.py:167-179,
 * and Kernel.matrix, kernels.py:75-93, inside M2LHandler.precompute,
 * m2l.py:136-273).  kernel 0 = Laplace 1/(4 pi r) (bit-identical to the host
 * assembly), 1 = Helmholtz exp(ikr)/(4 pi r).  nodes: HOST [n][3] reference
 * cube nodes (ChebyshevGrid.nodes3d); transfers: HOST int8 [n_t][3];
 * out: DEVICE [n_t][n][n] row-major, double (kernel 0) or interleaved
 * complex (kernel 1).  Enqueued on `stream` (NULL = default stream). */
int cfm_assemble_operators(int device, int kernel, double wavenumber, int n, const double* nodes, double width,
                           int n_t, const int8_t* transfers, double* out, void* stream);

/* The plan of the last cfm_apply_level_csr: cache_hit = 1 if it was reused
 * (plans of ad-hoc batches are cached under their exact CSR content, since
 * the reference's FmmPlan rebuilds identical batches on every run,
 * engine.py:98-120; they are kept apart from the level plans of
 * cfm_plan_level_*, which they never replace); mode 0 target tiles / 1 pair
 * entries; two_stage 1 for the two-stage low-rank plan; plan_id unique per
 * built plan (a cache hit returns the cached plan's id).  NULL outputs are
 * skipped. */
int cfm_last_csr_plan_info(cfm_handler* h, int* cache_hit, int* mode, int* two_stage, uint64_t* plan_id);

/* Device-side timing of the last apply (ms, CUDA events on the apply stream),
 * and the number of kernels it launched. */
int cfm_last_apply_stats(cfm_handler* h, double* ms, int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* CHEBM2L_H */
