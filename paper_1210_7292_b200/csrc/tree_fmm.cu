// GPU octree (octree.py:93-127) and the FMM stages around M2L (engine.py:122-199), operator assembly.
#include "internal.hpp"
#include "tree.cuh"
#include "fmm.cuh"
#include "precompute.cuh"
#include <cub/cub.cuh>

namespace cfm {

// ------------------------------------------------------------------ octree
struct TreeLevel {
  int64_t n = 0;
  DevBuf keys;  // sorted unique lexicographic keys
};

}  // namespace cfm

struct cfm_tree {
  int device = 0, depth = 0;
  int64_t n_points = 0;
  double center[3] = {0, 0, 0}, half = 1.0;
  std::vector<cfm::TreeLevel> levels;  // index = level
  cfm::DevBuf leaf_off, perm;          // leaf particle CSR (int64)
  cfm::DevBuf points;                  // n x 3 on the device (original order)
};

struct cfm_fmm {
  cfm_tree* tree = nullptr;
  int order = 0, n = 0;
  cfm::DevBuf troots, leaf_ijk, leaf_grid, leaf_of_pos;
  cfm::OpStack m2m_ops, l2l_ops;
  cfm::CodeMap octmap;
  std::map<int, cfm::LevelPlan> m2m_plans, l2l_plans;  // key: child level / parent level (x dc)
  // P2P: leaf-sorted positions (built on first use), sorted weights, leaf lists by size class
  cfm::DevBuf px, py, pz, sw, small_leaves, large_leaves;
  int64_t n_small = -1, n_large = 0;
};

namespace cfm {

template <class F>
static void cub_call(F&& f, cudaStream_t s) {
  size_t tmp = 0;
  CUDA_CHECK(f(nullptr, tmp));
  DevBuf t;
  t.alloc(std::max<size_t>(tmp, 16));
  CUDA_CHECK(f(t.p, tmp));
  CUDA_CHECK(cudaStreamSynchronize(s));
}

// sorted unique keys of `in` (n keys, device) -> out (device), returns count; optional run counts
static int64_t sort_unique(const unsigned long long* in, int64_t n, DevBuf& out, DevBuf* counts, int end_bit,
                           cudaStream_t s) {
  DevBuf sorted, nsel;
  sorted.alloc(std::max<size_t>(size_t(n) * 8, 16));
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, in, sorted.as<unsigned long long>(), int64_t(n), 0, end_bit, s);
  }, s);
  out.alloc(std::max<size_t>(size_t(n) * 8, 16));
  nsel.alloc(16);
  if (counts) {
    counts->alloc(std::max<size_t>(size_t(n) * 8, 16));
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRunLengthEncode::Encode(t, b, sorted.as<unsigned long long>(), out.as<unsigned long long>(),
                                                counts->as<long long>(), nsel.as<long long>(), int64_t(n), s);
    }, s);
  } else {
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceSelect::Unique(t, b, sorted.as<unsigned long long>(), out.as<unsigned long long>(),
                                       nsel.as<long long>(), int64_t(n), s);
    }, s);
  }
  long long m = 0;
  CUDA_CHECK(cudaMemcpy(&m, nsel.p, 8, cudaMemcpyDeviceToHost));
  return m;
}

static int key_bits(int level) { return std::max(1, 3 * level); }

}  // namespace cfm

using namespace cfm;

extern "C" {
int cfm_tree_build(int device, const double* points, int64_t n, const double* center, double half_width, int depth,
                   cfm_tree** out) {
  return guarded([&] {
    if (!out || !center) throw Error(CFM_ERR_VALUE, "null argument");
    if (depth < 2) throw Error(CFM_ERR_VALUE, "octree depth must be >= 2, got " + std::to_string(depth));
    if (depth > 20) throw Error(CFM_ERR_VALUE, "octree depth must be <= 20");
    if (n < 0) throw Error(CFM_ERR_VALUE, "negative particle count");
    if (!(half_width > 0)) throw Error(CFM_ERR_VALUE, "half_width must be positive");
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t s = nullptr;
    auto t = std::make_unique<cfm_tree>();
    t->device = device;
    t->depth = depth;
    t->n_points = n;
    t->levels.resize(depth + 1);
    for (int a = 0; a < 3; ++a) t->center[a] = center[a];
    t->half = half_width;
    t->points.alloc(std::max<size_t>(size_t(n) * 24, 16));
    if (n) CUDA_CHECK(cudaMemcpy(t->points.p, points, size_t(n) * 24, cudaMemcpyDefault));
    const double* dp = t->points.as<double>();
    DevBuf keys, idx, skeys, sidx, bad;
    keys.alloc(std::max<size_t>(size_t(n) * 8, 16));
    idx.alloc(std::max<size_t>(size_t(n) * 8, 16));
    bad.alloc(16);
    CUDA_CHECK(cudaMemset(bad.p, 0, 4));
    const double lx = center[0] - half_width, ly = center[1] - half_width, lz = center[2] - half_width;
    const double width = 2.0 * half_width;
    if (n) {
      k_leaf_keys<<<unsigned((n + 255) / 256), 256, 0, s>>>(dp, n, lx, ly, lz, width, depth,
                                                            keys.as<unsigned long long>(), idx.as<long long>(),
                                                            bad.as<int>());
      CUDA_CHECK(cudaGetLastError());
    }
    int hb = 0;
    CUDA_CHECK(cudaMemcpy(&hb, bad.p, 4, cudaMemcpyDeviceToHost));
    if (hb) throw Error(CFM_ERR_VALUE, "particle outside bounding box");
    // stable sort of (leaf key, particle index): particle indices ascend within a leaf
    skeys.alloc(std::max<size_t>(size_t(n) * 8, 16));
    sidx.alloc(std::max<size_t>(size_t(n) * 8, 16));
    t->perm.alloc(std::max<size_t>(size_t(n) * 8, 16));
    if (n) {
      cub_call([&](void* tp, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(tp, b, keys.as<unsigned long long>(), skeys.as<unsigned long long>(),
                                               idx.as<long long>(), t->perm.as<long long>(), int64_t(n), 0,
                                               key_bits(depth), s);
      }, s);
    }
    // leaves: unique keys and run lengths -> CSR offsets
    DevBuf counts;
    TreeLevel& leaf = t->levels[depth];
    leaf.n = n ? sort_unique(skeys.as<unsigned long long>(), n, leaf.keys, &counts, key_bits(depth), s) : 0;
    std::vector<long long> hc(leaf.n), ho(leaf.n + 1, 0);
    if (leaf.n) CUDA_CHECK(cudaMemcpy(hc.data(), counts.p, size_t(leaf.n) * 8, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < leaf.n; ++i) ho[i + 1] = ho[i] + hc[i];
    upload(t->leaf_off, ho);
    // coarser levels: sorted unique parents
    for (int L = depth; L >= 1; --L) {
      const TreeLevel& c = t->levels[L];
      TreeLevel& pl = t->levels[L - 1];
      if (c.n == 0) {
        pl.n = 0;
        continue;
      }
      DevBuf par;
      par.alloc(size_t(c.n) * 8);
      k_parent_keys<<<unsigned((c.n + 255) / 256), 256, 0, s>>>(c.keys.as<unsigned long long>(), c.n, 1ll << L,
                                                                par.as<unsigned long long>());
      CUDA_CHECK(cudaGetLastError());
      pl.n = sort_unique(par.as<unsigned long long>(), c.n, pl.keys, nullptr, key_bits(L - 1), s);
    }
    *out = t.release();
  });
}

int cfm_tree_level_size(cfm_tree* t, int level, int64_t* n_cells) {
  return guarded([&] {
    if (!t || !n_cells) throw Error(CFM_ERR_VALUE, "null argument");
    if (level < 0 || level > t->depth) throw Error(CFM_ERR_VALUE, "level outside the tree");
    *n_cells = t->levels[level].n;
  });
}

int cfm_tree_level_cells(cfm_tree* t, int level, int32_t* ijk_out) {
  return guarded([&] {
    if (!t || !ijk_out) throw Error(CFM_ERR_VALUE, "null argument");
    if (level < 0 || level > t->depth) throw Error(CFM_ERR_VALUE, "level outside the tree");
    CUDA_CHECK(cudaSetDevice(t->device));
    const TreeLevel& L = t->levels[level];
    if (!L.n) return;
    const bool dev = is_device_ptr(ijk_out);
    DevBuf tmp;
    int* d = ijk_out;
    if (!dev) {
      tmp.alloc(size_t(L.n) * 12);
      d = tmp.as<int>();
    }
    k_keys_to_ijk<<<unsigned((L.n + 255) / 256), 256>>>(L.keys.as<unsigned long long>(), L.n, 1ll << level, d);
    CUDA_CHECK(cudaGetLastError());
    if (!dev) CUDA_CHECK(cudaMemcpy(ijk_out, d, size_t(L.n) * 12, cudaMemcpyDeviceToHost));
    CUDA_CHECK(cudaDeviceSynchronize());
  });
}

int cfm_tree_leaf_particles(cfm_tree* t, int64_t* offsets_out, int64_t* perm_out) {
  return guarded([&] {
    if (!t) throw Error(CFM_ERR_VALUE, "null argument");
    CUDA_CHECK(cudaSetDevice(t->device));
    const int64_t nl = t->levels[t->depth].n;
    if (offsets_out)
      CUDA_CHECK(cudaMemcpy(offsets_out, t->leaf_off.p, size_t(nl + 1) * 8, cudaMemcpyDefault));
    if (perm_out && t->n_points)
      CUDA_CHECK(cudaMemcpy(perm_out, t->perm.p, size_t(t->n_points) * 8, cudaMemcpyDefault));
  });
}

int cfm_tree_destroy(cfm_tree* t) {
  return guarded([&] {
    if (!t) return;
    cudaSetDevice(t->device);
    delete t;
  });
}

// ---------------------------------------------------------------- FMM stages
static FmmGeom fmm_geom(cfm_fmm* f) {
  FmmGeom g{};
  cfm_tree* t = f->tree;
  g.pts = t->points.as<double>();
  g.perm = t->perm.as<long long>();
  g.leaf_off = t->leaf_off.as<long long>();
  g.leaf_ijk = f->leaf_ijk.as<int>();
  g.n_leaves = t->levels[t->depth].n;
  g.depth = t->depth;
  g.lx = t->center[0] - t->half;
  g.ly = t->center[1] - t->half;
  g.lz = t->center[2] - t->half;
  g.leaf_w = 2.0 * t->half / double(1ll << t->depth);
  g.troots = f->troots.as<double>();
  g.order = f->order;
  return g;
}

static std::vector<unsigned long long> host_keys(cfm_tree* t, int level) {
  std::vector<unsigned long long> k(t->levels[level].n);
  if (!k.empty())
    CUDA_CHECK(cudaMemcpy(k.data(), t->levels[level].keys.p, k.size() * 8, cudaMemcpyDeviceToHost));
  return k;
}

// M2M (child level L -> parent L-1) or L2L (parent L-1 -> child L) plan
static LevelPlan& fmm_plan(cfm_fmm* f, int child_level, bool up, int dc) {
  auto& plans = up ? f->m2m_plans : f->l2l_plans;
  const int key = child_level * 4 + dc;
  auto it = plans.find(key);
  if (it != plans.end()) return it->second;
  cfm_tree* t = f->tree;
  auto ck = host_keys(t, child_level);
  auto pk = host_keys(t, child_level - 1);
  const long long cs = 1ll << child_level, ps = cs >> 1;
  const int64_t nc = int64_t(ck.size()), np_ = int64_t(pk.size());
  std::vector<int64_t> parent(nc);
  std::vector<int16_t> oct(nc);
  for (int64_t c = 0; c < nc; ++c) {
    const long long z = ck[c] % cs, y = (ck[c] / cs) % cs, x = ck[c] / (cs * cs);
    const unsigned long long pkey = (unsigned long long)(((x >> 1) * ps + (y >> 1)) * ps + (z >> 1));
    parent[c] = int64_t(std::lower_bound(pk.begin(), pk.end(), pkey) - pk.begin());
    oct[c] = int16_t((x & 1) * 4 + (y & 1) * 2 + (z & 1));
  }
  std::vector<int64_t> tgt, off(1, 0), src;
  std::vector<int16_t> codes;
  if (up) {  // targets = parents, pairs = their children in octant (lexicographic) order
    std::vector<int64_t> ord(nc);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
      return parent[a] != parent[b] ? parent[a] < parent[b] : oct[a] < oct[b];
    });
    for (int64_t i = 0; i < nc;) {
      int64_t j = i;
      tgt.push_back(parent[ord[i]]);
      while (j < nc && parent[ord[j]] == parent[ord[i]]) {
        src.push_back(ord[j]);
        codes.push_back(oct[ord[j]]);
        ++j;
      }
      off.push_back(int64_t(src.size()));
      i = j;
    }
  } else {  // targets = children, one pair each: (parent, octant)
    for (int64_t c = 0; c < nc; ++c) {
      tgt.push_back(c);
      src.push_back(parent[c]);
      codes.push_back(oct[c]);
      off.push_back(int64_t(src.size()));
    }
  }
  std::array<int, kNumCodes> opkey;
  opkey.fill(-1);
  for (int c = 0; c < 8; ++c) opkey[c] = c;
  LevelPlan lp;
  try {
    lp.hp = build_plan_csr(int64_t(tgt.size()), tgt.data(), off.data(), src.data(), codes.data(), dc, opkey,
                           std::max(nc, np_));
  } catch (const PlanError& e) {
    throw Error(CFM_ERR_VALUE, e.what());
  }
  lp.dc = dc;
  lp.n_rows = std::max(nc, np_);
  push_plan(lp.hp, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src);
  plans[key] = std::move(lp);
  return plans[key];
}

static void fmm_shift(cfm_fmm* f, int child_level, bool up, const double* x, double* y, int data_complex,
                      cudaStream_t s) {
  if (child_level < 1 || child_level > f->tree->depth) throw Error(CFM_ERR_VALUE, "level outside the tree");
  const int dc = data_complex ? 2 : 1;
  LevelPlan& lp = fmm_plan(f, child_level, up, dc);
  TileParams p{};
  fill_ops(p, up ? f->m2m_ops : f->l2l_ops, f->octmap);
  fill_plan(p, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src, lp.hp.n_tiles);
  const long long row_ld = (long long)f->n * dc;
  p.x = x; p.x_ld = row_ld; p.x_dc = dc;
  p.y = y; p.y_ld = row_ld; p.y_dc = dc;
  p.scale = 1.0; p.accumulate = 1;
  launch_tiles(p, lp.hp.n_tiles, s);
}

int cfm_fmm_create(cfm_tree* t, int order, const double* shift_mats, cfm_fmm** out) {
  return guarded([&] {
    if (!t || !out || !shift_mats) throw Error(CFM_ERR_VALUE, "null argument");
    if (order < 2 || order > kMaxOrder) throw Error(CFM_ERR_VALUE, "order must be in [2, 12]");
    if (t->depth > 9) throw Error(CFM_ERR_VALUE, "FMM stages support depth <= 9");
    CUDA_CHECK(cudaSetDevice(t->device));
    auto f = std::make_unique<cfm_fmm>();
    f->tree = t;
    f->order = order;
    f->n = order * order * order;
    const int n = f->n;
    // T_k(root_i), k = 1..l-1 (interp.py:88-103 at the roots)
    std::vector<double> roots(order), tr(size_t(order) * (order - 1));
    const int half = order / 2;
    for (int i = 1; i <= half; ++i) roots[i - 1] = std::cos((2 * i - 1) * M_PI / (2 * order));
    if (order % 2) roots[half] = 0.0;
    for (int i = 0; i < half; ++i) roots[order - half + i] = -roots[half - 1 - i];
    for (int i = 0; i < order; ++i) {
      const double x = roots[i];
      double tm2 = 0, tm1 = 0;
      for (int k = 0; k < order - 1; ++k) {
        double v = (k == 0) ? x : (k == 1 ? 2.0 * x * x - 1.0 : 2.0 * x * tm1 - tm2);
        tr[size_t(i) * (order - 1) + k] = v;
        tm2 = tm1;
        tm1 = v;
      }
    }
    upload(f->troots, tr);
    const int64_t nl = t->levels[t->depth].n;
    f->leaf_ijk.alloc(std::max<size_t>(size_t(nl) * 12, 16));
    if (nl) {
      k_keys_to_ijk<<<unsigned((nl + 255) / 256), 256>>>(t->levels[t->depth].keys.as<unsigned long long>(), nl,
                                                          1ll << t->depth, f->leaf_ijk.as<int>());
      CUDA_CHECK(cudaGetLastError());
    }
    const long long S = 1ll << t->depth;
    f->leaf_grid.alloc(size_t(S * S * S) * sizeof(int));
    CUDA_CHECK(cudaMemset(f->leaf_grid.p, 0xff, f->leaf_grid.bytes));
    if (nl) k_leaf_grid<<<unsigned((nl + 255) / 256), 256>>>(f->leaf_ijk.as<int>(), nl, int(S), f->leaf_grid.as<int>());
    f->leaf_of_pos.alloc(std::max<size_t>(size_t(t->n_points) * 8, 16));
    if (nl) k_leaf_of_pos<<<unsigned((nl + 255) / 256), 256>>>(t->leaf_off.as<long long>(), nl, f->leaf_of_pos.as<long long>());
    CUDA_CHECK(cudaGetLastError());
    // M2M operators: mat (parent x child) per octant; L2L: transposes
    make_stack(f->m2m_ops, 8, n, n);
    make_stack(f->l2l_ops, 8, n, n);
    std::vector<double> blk(f->m2m_ops.stride), blt(f->l2l_ops.stride);
    for (int o = 0; o < 8; ++o) {
      std::fill(blk.begin(), blk.end(), 0.0);
      std::fill(blt.begin(), blt.end(), 0.0);
      const double* m = shift_mats + size_t(o) * n * n;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          blk[size_t(i) * f->m2m_ops.ld + j] = m[size_t(i) * n + j];
          blt[size_t(j) * f->l2l_ops.ld + i] = m[size_t(i) * n + j];
        }
      put_stack(f->m2m_ops, o, blk);
      put_stack(f->l2l_ops, o, blt);
    }
    for (int c = 0; c < 8; ++c) f->octmap.op[c] = c;
    f->octmap.push();
    CUDA_CHECK(cudaDeviceSynchronize());
    *out = f.release();
  });
}

int cfm_fmm_destroy(cfm_fmm* f) {
  return guarded([&] {
    if (!f) return;
    cudaSetDevice(f->tree->device);
    delete f;
  });
}

int cfm_fmm_p2m(cfm_fmm* f, const double* weights, int data_complex, double* leaf_mpoles, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    const int dc = data_complex ? 2 : 1;
    FmmGeom g = fmm_geom(f);
    if (!g.n_leaves) return;
    constexpr int CH = 64;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned nb = unsigned(g.n_leaves);
    const long long ld = (long long)f->n * dc;
    switch (f->order) {
      case 3: k_p2m_t<3, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 4: k_p2m_t<4, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 5: k_p2m_t<5, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 6: k_p2m_t<6, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 7: k_p2m_t<7, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 8: k_p2m_t<8, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      case 9: k_p2m_t<9, CH><<<nb, 128, 0, st>>>(g, weights, dc, leaf_mpoles, ld); break;
      default: {
        const int threads = f->n <= 1024 ? 128 : 256;
        const size_t smem = size_t(3 * f->order * CH + CH * 2) * sizeof(double);
        k_p2m<CH><<<nb, threads, smem, st>>>(g, weights, dc, leaf_mpoles, ld);
      }
    }
    CUDA_CHECK(cudaGetLastError());
  });
}

int cfm_fmm_m2m(cfm_fmm* f, int child_level, const double* child, double* parent, int data_complex, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    fmm_shift(f, child_level, true, child, parent, data_complex, static_cast<cudaStream_t>(stream));
  });
}

int cfm_fmm_l2l(cfm_fmm* f, int parent_level, const double* parent, double* child, int data_complex, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    fmm_shift(f, parent_level + 1, false, parent, child, data_complex, static_cast<cudaStream_t>(stream));
  });
}

int cfm_fmm_l2p(cfm_fmm* f, const double* leaf_locals, int data_complex, double* potentials, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    const int dc = data_complex ? 2 : 1;
    FmmGeom g = fmm_geom(f);
    const long long np_ = f->tree->n_points;
    if (!np_) return;
    const unsigned nb = unsigned((np_ + 127) / 128);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long* lop = f->leaf_of_pos.as<long long>();
    const long long ld = (long long)f->n * dc;
    switch (f->order) {
      case 3: k_l2p_t<3><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 4: k_l2p_t<4><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 5: k_l2p_t<5><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 6: k_l2p_t<6><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 7: k_l2p_t<7><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 8: k_l2p_t<8><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      case 9: k_l2p_t<9><<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_); break;
      default: k_l2p<<<nb, 128, 0, st>>>(g, lop, leaf_locals, ld, dc, potentials, np_);
    }
    CUDA_CHECK(cudaGetLastError());
  });
}

int cfm_fmm_p2p(cfm_fmm* f, int kernel, double wavenumber, const double* weights, int weights_complex,
                double* potentials, int out_complex, void* stream) {
  return guarded([&] {
    if (!f) throw Error(CFM_ERR_VALUE, "null handle");
    if (kernel != 0 && kernel != 1) throw Error(CFM_ERR_VALUE, "kernel must be 0 (Laplace) or 1 (Helmholtz)");
    if (weights_complex && !out_complex) throw Error(CFM_ERR_VALUE, "complex weights need complex potentials");
    if (kernel == 1 && !out_complex) throw Error(CFM_ERR_VALUE, "Helmholtz potentials are complex");
    CUDA_CHECK(cudaSetDevice(f->tree->device));
    FmmGeom g = fmm_geom(f);
    if (!g.n_leaves) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long np_ = f->tree->n_points;
    const unsigned nb = unsigned((np_ + 255) / 256);
    if (f->n_small < 0) {
      // leaf-sorted positions and the two leaf-size classes (<= 64 particles, more)
      f->px.alloc(std::max<size_t>(size_t(np_) * 8, 16));
      f->py.alloc(std::max<size_t>(size_t(np_) * 8, 16));
      f->pz.alloc(std::max<size_t>(size_t(np_) * 8, 16));
      if (np_) k_p2p_sort_pos<<<nb, 256, 0, st>>>(g.pts, g.perm, np_, f->px.as<double>(), f->py.as<double>(),
                                                    f->pz.as<double>());
      CUDA_CHECK(cudaGetLastError());
      std::vector<long long> off(size_t(g.n_leaves) + 1);
      CUDA_CHECK(cudaMemcpy(off.data(), g.leaf_off, off.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<long long> sm, lg;
      for (long long l = 0; l < g.n_leaves; ++l) (off[l + 1] - off[l] <= 64 ? sm : lg).push_back(l);
      upload(f->small_leaves, sm);
      upload(f->large_leaves, lg);
      f->n_small = int64_t(sm.size());
      f->n_large = int64_t(lg.size());
    }
    const int wdc = weights_complex ? 2 : 1;
    f->sw.alloc(std::max<size_t>(size_t(np_) * wdc * 8, 16));
    if (np_) {
      if (wdc == 2) k_p2p_sort_w<2><<<nb, 256, 0, st>>>(weights, g.perm, np_, f->sw.as<double>());
      else k_p2p_sort_w<1><<<nb, 256, 0, st>>>(weights, g.perm, np_, f->sw.as<double>());
      CUDA_CHECK(cudaGetLastError());
    }
    P2PGeom pg{g.leaf_off, g.leaf_ijk, f->leaf_grid.as<int>(), 1 << g.depth, f->px.as<double>(), f->py.as<double>(),
               f->pz.as<double>(), g.perm};
    auto run = [&](auto ker, auto wd, auto od) {
      constexpr int K = decltype(ker)::value, W = decltype(wd)::value, O = decltype(od)::value;
      if (f->n_small)
        k_p2p_small<K, W, O><<<unsigned(f->n_small), 128, 0, st>>>(pg, f->small_leaves.as<long long>(),
                                                                  f->sw.as<double>(), wavenumber, potentials);
      if (f->n_large)
        k_p2p_large<K, W, O><<<unsigned(f->n_large), 128, 0, st>>>(pg, f->large_leaves.as<long long>(),
                                                                  f->sw.as<double>(), wavenumber, potentials);
      CUDA_CHECK(cudaGetLastError());
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    if (kernel == 0 && wdc == 1 && !out_complex) run(I0{}, I1{}, I1{});
    else if (kernel == 0 && wdc == 1) run(I0{}, I1{}, I2{});
    else if (kernel == 0) run(I0{}, I2{}, I2{});
    else if (wdc == 1) run(I1{}, I1{}, I2{});
    else run(I1{}, I2{}, I2{});
  });
}

int cfm_assemble_operators(int device, int kernel, double wavenumber, int n, const double* nodes, double width,
                           int n_t, const int8_t* transfers, double* out, void* stream) {
  return guarded([&] {
    if (kernel != 0 && kernel != 1) throw Error(CFM_ERR_VALUE, "kernel must be 0 (Laplace) or 1 (Helmholtz)");
    if (n <= 0 || n > 2048 || n_t < 0) throw Error(CFM_ERR_VALUE, "bad operator size");
    if (!(width > 0.0)) throw Error(CFM_ERR_VALUE, "cell width must be positive");
    if (n_t == 0) return;
    if (!nodes || !transfers || !out) throw Error(CFM_ERR_VALUE, "null pointer");
    for (int t = 0; t < n_t; ++t) {
      const int a = transfers[3 * t], b = transfers[3 * t + 1], c = transfers[3 * t + 2];
      if (a * a + b * b + c * c <= 3) throw Error(CFM_ERR_VALUE, "transfer vector is not admissible (|t| <= sqrt(3))");
    }
    CUDA_CHECK(cudaSetDevice(device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DevBuf dn, dt;
    dn.alloc(size_t(n) * 3 * sizeof(double));
    dt.alloc(size_t(n_t) * 3);
    CUDA_CHECK(cudaMemcpyAsync(dn.p, nodes, size_t(n) * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(dt.p, transfers, size_t(n_t) * 3, cudaMemcpyHostToDevice, st));
    const long long nn = (long long)n * n;
    dim3 grid(unsigned((nn + 255) / 256), unsigned(n_t));
    k_assemble<<<grid, 256, size_t(n) * 3 * sizeof(double), st>>>(kernel, wavenumber, n, dn.as<double>(), width,
                                                                 dt.as<int8_t>(), out);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaStreamSynchronize(st));  // the staging buffers are freed on return
  });
}

}  // extern "C"
