// Operator cache: permutation tables, full-operator / low-rank / two-stage stacks (m2l.py:136-273 on the device).
#include "internal.hpp"

namespace cfm {

// ------------------------------------------------------------------ handler ops
void build_tables(cfm_handler* h) {
  const int nf = h->n * h->f;
  std::vector<int16_t> row(size_t(kNumPerms) * nf), inv(size_t(kNumPerms) * nf);
  for (int pid = 0; pid < kNumPerms; ++pid) {
    auto tab = permutation_table(pid, h->order);
    auto itab = inverse_table(tab);
    for (int i = 0; i < h->n; ++i)
      for (int q = 0; q < h->f; ++q) {
        row[size_t(pid) * nf + i * h->f + q] = int16_t(tab[i] * h->f + q);
        inv[size_t(pid) * nf + i * h->f + q] = int16_t(itab[i] * h->f + q);
      }
  }
  upload(h->rowtab, row);
  upload(h->invtab, inv);
}

// Map every transfer of the group to (op index, perm) following the variant:
// symmetric variants go through canonicalize (symmetry.py:63-75, lookup :142-144),
// plain ones index the operator of t itself.
void map_transfers(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers, int n_ops,
                          const int8_t* op_t, bool rows_permuted, bool cols_permuted, CodeMap& m) {
  std::array<int, kNumCodes> op_of_code;
  op_of_code.fill(-1);
  for (int i = 0; i < n_ops; ++i) {
    const int t0 = op_t[3 * i], t1 = op_t[3 * i + 1], t2 = op_t[3 * i + 2];
    if (t0 < -3 || t0 > 3 || t1 < -3 || t1 > 3 || t2 < -3 || t2 > 3)
      throw Error(CFM_ERR_VALUE, "operator transfer vector outside [-3,3]^3");
    op_of_code[tcode(t0, t1, t2)] = i;
  }
  for (int k = 0; k < n_transfers; ++k) {
    const int t0 = transfers[3 * k], t1 = transfers[3 * k + 1], t2 = transfers[3 * k + 2];
    if (t0 < -3 || t0 > 3 || t1 < -3 || t1 > 3 || t2 < -3 || t2 > 3)
      throw Error(CFM_ERR_VALUE, "transfer vector outside [-3,3]^3");
    const int c = tcode(t0, t1, t2);
    g.valid[c] = 1;
    if (h->sym) {
      int ts[3], pid;
      canonicalize(t0, t1, t2, ts, pid);
      const int o = op_of_code[tcode(ts[0], ts[1], ts[2])];
      if (o < 0) throw Error(CFM_ERR_PRECOMPUTE, "no representative operator for a transfer vector");
      m.op[c] = o;
      m.rperm[c] = rows_permuted ? pid : -1;
      m.cperm[c] = cols_permuted ? pid : -1;
    } else {
      const int o = op_of_code[c];
      if (o < 0) throw Error(CFM_ERR_PRECOMPUTE, "no operator for a transfer vector");
      m.op[c] = o;
    }
  }
}


// Full-operator stack for the TMA tile kernel: K_t[i][j] = Op[tab_r[i]][tab_c[j]]
// for every transfer of the group (the same products the permuted apply forms,
// acc[i] += sum_k Op[rowtab[i]][k] x[invtab[k]] with j = invtab[k]), rows padded
// to a multiple of 8, columns to the KC multiple; plus the 2-D tensor map.
void build_full_ops(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers, const double* ops) {
  const int n = h->n;
  const int rows = round_up(n, 8);
  OpStack& fs = g.full;
  make_stack(fs, n_transfers, rows, n);
  g.full_rows = rows;
  std::vector<double> blockv(fs.stride);
  std::vector<int> ident(n);
  std::iota(ident.begin(), ident.end(), 0);
  for (int k = 0; k < n_transfers; ++k) {
    const int c = tcode(transfers[3 * k], transfers[3 * k + 1], transfers[3 * k + 2]);
    const int o = g.main.op[c], rp = g.main.rperm[c], cp = g.main.cperm[c];
    const std::vector<int> tr = rp >= 0 ? permutation_table(rp, h->order) : ident;
    const std::vector<int> tc = cp >= 0 ? permutation_table(cp, h->order) : ident;
    std::fill(blockv.begin(), blockv.end(), 0.0);
    const double* src = ops + size_t(o) * n * n;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) blockv[size_t(i) * fs.ld + j] = src[size_t(tr[i]) * n + tc[j]];
    put_stack(fs, k, blockv);
    g.fullmap.op[c] = k;
  }
  g.fullmap.push();
  const cuuint64_t dims[2] = {cuuint64_t(fs.ld), cuuint64_t(n_transfers) * rows};
  const cuuint64_t strides[1] = {cuuint64_t(fs.ld) * sizeof(double)};
  const cuuint32_t box[2] = {cuuint32_t(kKC + 4), 128u};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = resolve_encode_tiled()(&g.full_tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, fs.d.p, dims, strides,
                                            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuTensorMapEncodeTiled failed for the operator stack");
  g.has_full = true;
}

void make_stack(OpStack& s, int n_ops, int rows, int cols) {
  s.n_ops = n_ops;
  s.rows = rows;
  s.cols = cols;
  s.ld = round_up(std::max(cols, 1), kKC);
  s.stride = (long long)rows * s.ld;
  s.d.alloc(std::max<size_t>(size_t(n_ops) * s.stride * sizeof(double), 16));
  CUDA_CHECK(cudaMemset(s.d.p, 0, s.d.bytes));
}

void put_stack(OpStack& s, int i, const std::vector<double>& hostblock) {
  CUDA_CHECK(cudaMemcpy(s.d.as<double>() + (size_t)i * s.stride, hostblock.data(),
                        hostblock.size() * sizeof(double), cudaMemcpyHostToDevice));
}

void set_per_op(OpStack& s, const std::vector<int>& rows, const std::vector<int>& klen) {
  if (!rows.empty()) {
    upload(s.d_rows, rows);
    s.has_rows = true;
  }
  if (!klen.empty()) {
    upload(s.d_klen, klen);
    s.has_klen = true;
  }
}

// Low-rank factor stacks: pass 1 op = right^H (r f x n f), pass 2 op = left (n f x r f).
void build_lowrank_stacks(cfm_handler* h, OpStack& left, OpStack& right_h, int n_ops, const int* ranks,
                                 const double* L, const double* R, int rows_left, int rows_right) {
  // rows_left: rows of left (n or r_u); rows_right: rows of right (n or r_b)
  const int f = h->f;
  const bool cplx = h->op_complex;
  int rmax = 0;
  for (int i = 0; i < n_ops; ++i) rmax = std::max(rmax, ranks[i]);
  make_stack(left, n_ops, rows_left * f, std::max(rmax * f, 1));
  make_stack(right_h, n_ops, std::max(rmax * f, 1), rows_right * f);
  std::vector<int> rrows(n_ops), rk(n_ops);
  size_t offL = 0, offR = 0;
  const int sc = cplx ? 2 : 1;
  for (int i = 0; i < n_ops; ++i) {
    const int r = ranks[i];
    rrows[i] = r * f;
    rk[i] = r * f;
    std::vector<double> bl((size_t)left.stride, 0.0), br((size_t)right_h.stride, 0.0);
    if (r > 0) {
      realify_into(L + offL, rows_left, r, cplx, bl.data(), left.ld);
      realify_into(R + offR, r, rows_right, cplx, br.data(), right_h.ld, /*conj_t=*/true);
    }
    put_stack(left, i, bl);
    put_stack(right_h, i, br);
    offL += (size_t)rows_left * r * sc;
    offR += (size_t)rows_right * r * sc;
    left.host_bytes += (size_t)rows_left * r * sc * 8;
    right_h.host_bytes += (size_t)rows_right * r * sc * 8;
  }
  set_per_op(left, {}, rk);       // pass 2: inner length = rank
  set_per_op(right_h, rrows, {});  // pass 1: rows = rank
}

// CFM_LR_TWOSTAGE: 0 off (fused kernel), 1 source-major Y with rank-segment
// stage 2 (round 1), 2 target-major Y with a dense stage 2 (default).  Read at
// every precompute and plan build (tests switch it).
int two_stage_mode() {
  const char* e = getenv("CFM_LR_TWOSTAGE");
  return e ? atoi(e) : 2;
}
bool use_two_stage() { return two_stage_mode() != 0; }

// Target-major two-stage stacks (Group::has_tsT).  Per class c (the 8 range
// patterns of octree far lists; a target's transfers fall in one of them just
// like a source's) its transfers k, ascending, own the packed rows
// [rho_T[c][k], rho_T[c][k] + r_k): the V stack of class c holds V_k^H there
// (stage 1, sources of class c), the U stack holds U_k's columns there (stage
// 2, targets of class c).
static void build_two_stage_target_major(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers,
                                         const std::vector<int>& rk, const std::vector<double>& all_v,
                                         const std::vector<double>& all_u) {
  g.has_tsT = false;
  const int n = h->n;
  g.tsT_rho.assign(size_t(8) * n_transfers, -1);
  g.tsT_slot.assign(size_t(8) * n_transfers, -1);
  g.tsT_nblk.assign(8, 0);
  int max_rows = 0, max_slots = 0;
  for (int cls = 0; cls < 8; ++cls) {
    int rows = 0, slots = 0;
    std::vector<int> members;
    for (int k = 0; k < n_transfers; ++k) {
      bool in = rk[k] > 0;
      for (int a = 0; a < 3 && in; ++a) {
        const int t = transfers[3 * k + a], bit = (cls >> a) & 1;
        in = t >= (bit ? -2 : -3) && t <= (bit ? 3 : 2);
      }
      if (in) members.push_back(k);
    }
    // slot order: transfers of equal component parities together, the last
    // component fastest.  Consecutive slots then mostly differ by 2 in the last
    // component, so for one target the two pairs' sources are same-class
    // neighbours along the fastest cell axis -- the same stage-1 tile --
    // and the 32-B sector their rank runs share in the target's Y_T row is
    // completed by one CTA instead of being evicted half written.
    auto key = [&](int k) {
      const int t0 = transfers[3 * k], t1 = transfers[3 * k + 1], t2 = transfers[3 * k + 2];
      const int par = ((t0 & 1) << 2) | ((t1 & 1) << 1) | (t2 & 1);
      return (((par * 8 + (t0 + 3)) * 8 + (t1 + 3)) * 8) + (t2 + 3);
    };
    std::sort(members.begin(), members.end(), [&](int a, int b) { return key(a) < key(b); });
    for (int k : members) {
      g.tsT_rho[size_t(cls) * n_transfers + k] = rows;
      g.tsT_slot[size_t(cls) * n_transfers + k] = slots++;
      rows += rk[k];
    }
    g.tsT_nblk[cls] = (rows + 127) / 128;
    max_rows = std::max(max_rows, rows);
    max_slots = std::max(max_slots, slots);
  }
  if (max_rows == 0 || max_slots >= (1 << 23)) return;
  const int nb = (max_rows + 127) / 128;
  g.tsT_nb = nb;
  g.tsT_nslots = max_slots;
  std::vector<int> rowinfo(size_t(8) * nb * 128, -1);
  for (int cls = 0; cls < 8; ++cls)
    for (int k = 0; k < n_transfers; ++k) {
      const int r0 = g.tsT_rho[size_t(cls) * n_transfers + k];
      if (r0 < 0) continue;
      const int slot = g.tsT_slot[size_t(cls) * n_transfers + k];
      for (int a = 0; a < rk[k]; ++a) rowinfo[size_t(cls) * nb * 128 + r0 + a] = (slot << 8) | a;
    }
  upload(g.tsT_rowinfo, rowinfo);
  const int urows = round_up(n, 8);
  make_stack(g.tsT_v, 8 * nb, 128, n);
  make_stack(g.tsT_u, 8 * nb, urows, 128);
  const int vld = g.lrf_right_h.ld, uld = g.lrf_left.ld;
  const size_t vstride = size_t(g.lrf_right_h.stride), ustride = size_t(g.lrf_left.stride);
  std::vector<double> vb(size_t(g.tsT_v.stride)), ub(size_t(g.tsT_u.stride));
  for (int cls = 0; cls < 8; ++cls)
    for (int b = 0; b < nb; ++b) {
      std::fill(vb.begin(), vb.end(), 0.0);
      std::fill(ub.begin(), ub.end(), 0.0);
      for (int k = 0; k < n_transfers; ++k) {
        const int r0 = g.tsT_rho[size_t(cls) * n_transfers + k];
        if (r0 < 0) continue;
        for (int a = 0; a < rk[k]; ++a) {
          const int row = r0 + a;
          if (row / 128 != b) continue;
          std::copy_n(all_v.begin() + size_t(k) * vstride + size_t(a) * vld, n,
                      vb.begin() + size_t(row % 128) * g.tsT_v.ld);
          for (int i = 0; i < n; ++i)
            ub[size_t(i) * g.tsT_u.ld + row % 128] = all_u[size_t(k) * ustride + size_t(i) * uld + a];
        }
      }
      put_stack(g.tsT_v, cls * nb + b, vb);
      put_stack(g.tsT_u, cls * nb + b, ub);
    }
  auto encode = [](CUtensorMap* m, const OpStack& st, long long rows) {
    const cuuint64_t dims[2] = {cuuint64_t(st.ld), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(st.ld) * sizeof(double)};
    const cuuint32_t box[2] = {cuuint32_t(kKC + 4), 128u};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = resolve_encode_tiled()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, st.d.p, dims, strides, box, estr,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuTensorMapEncodeTiled failed for a target-major two-stage stack");
  };
  encode(&g.tsT_vmap, g.tsT_v, (long long)8 * nb * 128);
  encode(&g.tsT_umap, g.tsT_u, (long long)8 * nb * urows);
  g.has_tsT = true;
}

// Two-stage low-rank operators (see Group::has_ts): per source class the V_t^H
// rows of its transfers packed back to back (transfer k's r_k rows start at
// ts_rho0[cls][k], rounded up to 4 rows = one stage-2 k-step), so stage 1
// computes sum_k ceil4(r_k) rows per source instead of 16-row segments
// (l = 5, eps = 1e-5: 20 row blocks of 128 instead of 26).  Stage 1 writes a
// source's rows to Y[source][ycol[k] + a] (ts_colmap), one column range per
// transfer for all classes: stage 2 gathers an entry's B at column
// ycol[k] + 16 j (ts_opcol; 32-B aligned) whatever its sources' classes.
void build_two_stage(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers,
                     const std::vector<int>& rk, const std::vector<double>& all_v, const std::vector<double>& all_u) {
  g.has_ts = false;
  g.has_tsT = false;
  if (!use_two_stage()) return;
  const int n = h->n;
  int rmax = 0;
  for (int r : rk) rmax = std::max(rmax, r);
  if (rmax == 0 || rmax > 255 || n > 1024) return;
  g.ts_ntr = n_transfers;
  g.ts_rank = rk;
  if (two_stage_mode() >= 2) build_two_stage_target_major(h, g, n_transfers, transfers, rk, all_v, all_u);
  if (rmax > 32 || g.lrf_left.ld != 32) return;
  g.ts_rho0.assign(size_t(8) * n_transfers, -1);
  int max_rows = 0;
  for (int cls = 0; cls < 8; ++cls) {
    int rows = 0;
    for (int k = 0; k < n_transfers; ++k) {
      bool in = rk[k] > 0;
      for (int a = 0; a < 3 && in; ++a) {
        const int t = transfers[3 * k + a], bit = (cls >> a) & 1;
        in = t >= (bit ? -2 : -3) && t <= (bit ? 3 : 2);
      }
      if (!in) continue;
      g.ts_rho0[size_t(cls) * n_transfers + k] = rows;
      rows += (rk[k] + 3) / 4 * 4;  // 32-B aligned starts: stage 2's gather column coordinates
    }
    max_rows = std::max(max_rows, rows);
  }
  const int nb = (max_rows + 127) / 128;
  g.ts_nb = nb;
  // Y columns: transfer k's ceil4(r_k) rows at the same column for every
  // class (a stage-2 entry's sources may sit in different classes)
  std::vector<int> ycol(n_transfers, -1);
  int ldy = 0;
  for (int k = 0; k < n_transfers; ++k)
    if (rk[k] > 0) {
      ycol[k] = ldy;
      ldy += (rk[k] + 3) / 4 * 4;
    }
  g.ts_ldy = ldy;
  std::vector<int> colmap(size_t(8) * nb * 128, -1);
  for (int cls = 0; cls < 8; ++cls)
    for (int k = 0; k < n_transfers; ++k) {
      const int r0 = g.ts_rho0[size_t(cls) * n_transfers + k];
      if (r0 < 0) continue;
      for (int a = 0; a < (rk[k] + 3) / 4 * 4; ++a) colmap[size_t(cls) * nb * 128 + r0 + a] = ycol[k] + a;
    }
  upload(g.ts_colmap, colmap);
  std::vector<int> opcol(size_t(2) * n_transfers, 0);
  for (int k = 0; k < n_transfers; ++k)
    for (int j = 0; j < 2; ++j) opcol[size_t(2) * k + j] = std::max(ycol[k], 0) + 16 * j;
  upload(g.ts_opcol, opcol);
  make_stack(g.ts_v, 8 * nb, 128, n);
  const int vld = g.lrf_right_h.ld;
  const size_t vstride = size_t(g.lrf_right_h.stride);
  std::vector<double> blk(size_t(g.ts_v.stride));
  for (int cls = 0; cls < 8; ++cls)
    for (int b = 0; b < nb; ++b) {
      std::fill(blk.begin(), blk.end(), 0.0);
      for (int k = 0; k < n_transfers; ++k) {
        const int r0 = g.ts_rho0[size_t(cls) * n_transfers + k];
        if (r0 < 0) continue;
        for (int a = 0; a < rk[k]; ++a) {
          const int row = r0 + a;
          if (row / 128 != b) continue;
          std::copy_n(all_v.begin() + size_t(k) * vstride + size_t(a) * vld, n,
                      blk.begin() + size_t(row % 128) * g.ts_v.ld);
        }
      }
      put_stack(g.ts_v, cls * nb + b, blk);
    }
  auto encode = [](CUtensorMap* m, const OpStack& st, long long rows, unsigned box0) {
    const cuuint64_t dims[2] = {cuuint64_t(st.ld), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(st.ld) * sizeof(double)};
    const cuuint32_t box[2] = {box0, 128u};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = resolve_encode_tiled()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, st.d.p, dims, strides, box, estr,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(CFM_ERR_CUDA, "cuTensorMapEncodeTiled failed for a two-stage stack");
  };
  encode(&g.ts_vmap, g.ts_v, (long long)8 * nb * 128, kKC + 4);
  encode(&g.ts_umap, g.lrf_left, (long long)n_transfers * n, 16 + 4);
  // stage 2 skips the k-steps of a 16-wide rank segment past the rank (in a
  // partial last k-step the U_t columns and Y rows past the rank are exact
  // zeros), so sums are unchanged
  std::vector<int> ks(size_t(2) * n_transfers, 0);
  for (int k = 0; k < n_transfers; ++k)
    for (int j = 0; j < 2; ++j) {
      const int w = std::min(16, std::max(0, rk[k] - 16 * j));
      ks[size_t(2) * k + j] = (w + 3) / 4;
    }
  upload(g.ts_ksteps, ks);
  g.has_ts = true;
}

// Per-transfer low-rank factors for real operators: U_t[i][a] = left_o[tab_r[i]][a],
// V_t^H[a][j] = right_o[tab_c[j]][a] (the products the permuted apply forms:
// Y[a] = sum_k right^H[a][k] x[inv[k]] = sum_j right^H[a][tab[j]] x[j]).
void build_lowrank_full(cfm_handler* h, Group& g, int n_transfers, const int8_t* transfers, int n_ops,
                               const int* ranks, const double* L, const double* R) {
  // Complex operators: the factors are realified first ([[Re, -Im], [Im, Re]] per
  // element, rows / columns interleaved like a complex128 expansion row), and a
  // permutation of the n coefficients moves the (re, im) row pairs together.
  const int n = h->n, f = h->f;
  const bool cplx = h->op_complex;
  const int nf = n * f, sc = cplx ? 2 : 1;
  int rmax = 0;
  for (int i = 0; i < n_ops; ++i) rmax = std::max(rmax, ranks[i]);
  std::vector<size_t> off(n_ops + 1, 0);
  for (int i = 0; i < n_ops; ++i) off[i + 1] = off[i] + size_t(n) * ranks[i] * sc;
  make_stack(g.lrf_left, n_transfers, nf, std::max(rmax * f, 1));
  make_stack(g.lrf_right_h, n_transfers, std::max(rmax * f, 1), nf);
  std::vector<int> ident(n), rk(n_transfers);
  std::iota(ident.begin(), ident.end(), 0);
  std::vector<double> bl(g.lrf_left.stride), br(g.lrf_right_h.stride);
  std::vector<double> tl(g.lrf_left.stride), tr_(g.lrf_right_h.stride);
  std::vector<double> all_v(size_t(n_transfers) * g.lrf_right_h.stride);
  std::vector<double> all_u(size_t(n_transfers) * g.lrf_left.stride);
  const int lld = g.lrf_left.ld, rld = g.lrf_right_h.ld;
  for (int k = 0; k < n_transfers; ++k) {
    const int c = tcode(transfers[3 * k], transfers[3 * k + 1], transfers[3 * k + 2]);
    const int o = g.main.op[c];
    const std::vector<int> tr = g.main.rperm[c] >= 0 ? permutation_table(g.main.rperm[c], h->order) : ident;
    const std::vector<int> tc = g.pass1.cperm[c] >= 0 ? permutation_table(g.pass1.cperm[c], h->order) : ident;
    const int r = ranks[o];
    rk[k] = r * f;
    std::fill(bl.begin(), bl.end(), 0.0);
    std::fill(br.begin(), br.end(), 0.0);
    if (r > 0) {
      std::fill(tl.begin(), tl.end(), 0.0);
      std::fill(tr_.begin(), tr_.end(), 0.0);
      realify_into(L + off[o], n, r, cplx, tl.data(), lld);                       // left: (n f) x (r f)
      realify_into(R + off[o], r, n, cplx, tr_.data(), rld, /*conj_t=*/true);      // right^H: (r f) x (n f)
      for (int i = 0; i < n; ++i)
        for (int q = 0; q < f; ++q)
          std::copy_n(tl.begin() + size_t(tr[i] * f + q) * lld, r * f, bl.begin() + size_t(i * f + q) * lld);
      for (int a = 0; a < r * f; ++a)
        for (int j = 0; j < n; ++j)
          for (int q = 0; q < f; ++q) br[size_t(a) * rld + j * f + q] = tr_[size_t(a) * rld + tc[j] * f + q];
    }
    put_stack(g.lrf_left, k, bl);
    put_stack(g.lrf_right_h, k, br);
    std::copy(br.begin(), br.end(), all_v.begin() + size_t(k) * br.size());
    std::copy(bl.begin(), bl.end(), all_u.begin() + size_t(k) * bl.size());
    g.fullmap.op[c] = k;
  }
  g.fullmap.push();
  set_per_op(g.lrf_left, {}, rk);
  set_per_op(g.lrf_right_h, rk, {});
  g.has_lrfull = true;
  if (PFN_encodeTiled enc = resolve_encode_tiled()) {
    auto encode = [&](CUtensorMap* m, const OpStack& st) {
      const cuuint64_t dims[2] = {cuuint64_t(st.ld), cuuint64_t((long long)st.n_ops * st.rows)};
      const cuuint64_t strides[1] = {cuuint64_t(st.ld) * sizeof(double)};
      const cuuint32_t box[2] = {cuuint32_t(kKC + 4), 128u};
      const cuuint32_t estr[2] = {1u, 1u};
      return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, st.d.p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    g.has_lrmaps = encode(&g.lrf_umap, g.lrf_left) && encode(&g.lrf_vmap, g.lrf_right_h);
  }
  if (!cplx) build_two_stage(h, g, n_transfers, transfers, rk, all_v, all_u);
}

}  // namespace cfm
