// Host plan builder: CSR far lists -> tiles x entries for tile_gemm_kernel.
//
// The reference applies a level's batch by walking each target's far list
// (m2l.py:320-364) or by filling 128-column buffers per cone representative
// and flushing them (m2l.py:397-452).  On the GPU the unit of work is a tile of
// BN output columns (targets, or (target, re/im) pairs for complex expansions
// under a real operator); for each tile the pairs are grouped by
// (operator, transfer vector, occurrence) into entries whose BN source
// columns share one operator and one permutation.  Targets are ordered so
// that tiles hold targets with identical transfer-vector multisets (same
// octant and boundary class on a full level), which makes every entry dense.
//
// Everything here is integer bookkeeping done once per (handler, level); the
// result is cached and uploaded.
#pragma once
#include <algorithm>
#include <array>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "symmetry.hpp"

namespace cfm {

constexpr int kBN = 64;

struct HostPlan {
  int bn = kBN;
  int dc = 1;
  int64_t n_tiles = 0;
  std::vector<int> tile_col;    // n_tiles * bn, virtual column ids (target_row*dc + comp) or -1
  std::vector<int> tile_off;    // n_tiles + 1
  std::vector<int> entry_code;  // E
  std::vector<int> entry_src;   // E * bn, virtual source ids or -1
  int64_t n_pairs = 0;
  std::array<int64_t, kNumCodes> code_count{};
  int64_t n_entries_dev = -1;  // >= 0: the arrays were built on the device only (plan_device.cu)
  int64_t n_entries() const { return n_entries_dev >= 0 ? n_entries_dev : int64_t(entry_code.size()); }
};

inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct PlanError : std::runtime_error {
  int code;
  PlanError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// opkey[code] >= 0 gives the operator the code maps to (entries are ordered by
// it, so that one operator's entries are contiguous inside a tile); a pair
// whose code has opkey < 0 has no precomputed operator.
inline HostPlan build_plan_csr(int64_t n_targets, const int64_t* tgt, const int64_t* off,
                               const int64_t* src, const int16_t* codes, int dc,
                               const std::array<int, kNumCodes>& opkey, int64_t n_rows,
                               int n_threads = 0) {
  HostPlan plan;
  plan.dc = dc;
  const int tpt = kBN / dc;  // targets per tile
  // 1. targets with pairs; merge duplicate target rows (rare; the engine never
  //    emits them, but apply_level accepts any batch)
  std::vector<int64_t> order;
  order.reserve(n_targets);
  for (int64_t i = 0; i < n_targets; ++i) {
    if (tgt[i] < 0 || tgt[i] >= n_rows) throw PlanError(1, "target row out of range");
    if (off[i + 1] < off[i]) throw PlanError(1, "offsets must be non-decreasing");
    if (off[i + 1] > off[i]) order.push_back(i);
  }
  // group batch entries by target row (stable)
  std::vector<int64_t> by_row(order);
  std::stable_sort(by_row.begin(), by_row.end(), [&](int64_t a, int64_t b) { return tgt[a] < tgt[b]; });
  // unique targets: first batch index, list of batch indices
  std::vector<int64_t> uniq_first;        // representative batch index (first occurrence)
  std::vector<int64_t> grp_start, grp_items;  // CSR over batch indices per unique target
  uniq_first.reserve(by_row.size());
  for (size_t i = 0; i < by_row.size();) {
    size_t j = i;
    int64_t first = by_row[i];
    grp_start.push_back(int64_t(grp_items.size()));
    while (j < by_row.size() && tgt[by_row[j]] == tgt[by_row[i]]) {
      first = std::min(first, by_row[j]);
      grp_items.push_back(by_row[j]);
      ++j;
    }
    uniq_first.push_back(first);
    i = j;
  }
  grp_start.push_back(int64_t(grp_items.size()));
  const int64_t nu = int64_t(uniq_first.size());

  unsigned nth = n_threads > 0 ? unsigned(n_threads) : std::max(1u, std::thread::hardware_concurrency());
  // 2. code-multiset hash per unique target (order independent), validity
  //    checks; parallel over unique targets (the first error in target order wins)
  std::vector<uint64_t> hash(nu, 0);
  {
    const unsigned nh = unsigned(std::min<int64_t>(nth, std::max<int64_t>(1, nu / 4096)));
    std::vector<int64_t> bad_u(nh, nu);
    std::vector<int> bad_kind(nh, 0), bad_code(nh, 0);
    auto hwork = [&](unsigned w) {
      for (int64_t u = int64_t(w) * nu / nh; u < int64_t(w + 1) * nu / nh; ++u) {
        uint64_t h = 0;
        for (int64_t gi = grp_start[u]; gi < grp_start[u + 1]; ++gi) {
          const int64_t b = grp_items[gi];
          for (int64_t q = off[b]; q < off[b + 1]; ++q) {
            const int c = codes[q];
            int kind = 0;
            if (c < 0 || c >= kNumCodes) kind = 1;
            else if (opkey[c] < 0) kind = 2;
            else if (src[q] < 0 || src[q] >= n_rows) kind = 3;
            if (kind) {
              bad_u[w] = u, bad_kind[w] = kind, bad_code[w] = c;
              return;
            }
            h += splitmix64(uint64_t(c) + 1);
          }
        }
        hash[u] = h;
      }
    };
    std::vector<std::thread> hp;
    for (unsigned w = 1; w < nh; ++w) hp.emplace_back(hwork, w);
    hwork(0);
    for (auto& th : hp) th.join();
    for (unsigned w = 0; w < nh; ++w) {
      if (bad_u[w] == nu) continue;
      if (bad_kind[w] == 1) throw PlanError(1, "transfer vector outside [-3,3]^3");
      if (bad_kind[w] == 3) throw PlanError(1, "source row out of range");
      int t0, t1, t2;
      tcode_decode(bad_code[w], t0, t1, t2);
      throw PlanError(2, "no operator for transfer vector (" + std::to_string(t0) + ", " + std::to_string(t1) +
                             ", " + std::to_string(t2) + ")");
    }
  }
  // 3. order: by hash, then by first appearance in the batch
  std::vector<int64_t> uord(nu);
  std::iota(uord.begin(), uord.end(), 0);
  std::sort(uord.begin(), uord.end(), [&](int64_t a, int64_t b) {
    if (hash[a] != hash[b]) return hash[a] < hash[b];
    return uniq_first[a] < uniq_first[b];
  });
  // 4. tiles
  const int64_t n_tiles = (nu + tpt - 1) / tpt;
  plan.n_tiles = n_tiles;
  plan.tile_col.assign(size_t(n_tiles) * kBN, -1);
  for (int64_t k = 0; k < nu; ++k) {
    const int64_t tile = k / tpt, slot = k % tpt;
    const int64_t row = tgt[uniq_first[uord[k]]];
    for (int q = 0; q < dc; ++q) plan.tile_col[size_t(tile) * kBN + slot * dc + q] = int(row * dc + q);
  }
  // 5. entries per tile (parallel over tiles)
  std::vector<std::vector<int>> t_code(n_tiles), t_src(n_tiles);
  std::vector<std::array<int64_t, kNumCodes>> part_count;
  nth = unsigned(std::min<int64_t>(nth, std::max<int64_t>(1, n_tiles / 64)));
  part_count.resize(nth);
  auto work = [&](unsigned w) {
    auto& cc = part_count[w];
    cc.fill(0);
    struct Item {
      int key, code, occ, slot, src;
    };
    std::vector<Item> items;
    std::vector<int> occ_cnt(kNumCodes, 0);
    std::vector<int> touched;
    for (int64_t tile = w; tile < n_tiles; tile += nth) {
      items.clear();
      for (int s = 0; s < tpt; ++s) {
        const int64_t k = tile * tpt + s;
        if (k >= nu) break;
        const int64_t u = uord[k];
        touched.clear();
        for (int64_t gi = grp_start[u]; gi < grp_start[u + 1]; ++gi) {
          const int64_t b = grp_items[gi];
          for (int64_t q = off[b]; q < off[b + 1]; ++q) {
            const int c = codes[q];
            if (occ_cnt[c] == 0) touched.push_back(c);
            items.push_back({opkey[c], c, occ_cnt[c]++, s, int(src[q])});
            cc[c] += 1;
          }
        }
        for (int c : touched) occ_cnt[c] = 0;
      }
      std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
        if (a.key != b.key) return a.key < b.key;
        if (a.code != b.code) return a.code < b.code;
        if (a.occ != b.occ) return a.occ < b.occ;
        return a.slot < b.slot;
      });
      auto& codes_out = t_code[tile];
      auto& src_out = t_src[tile];
      for (size_t i = 0; i < items.size();) {
        size_t j = i;
        codes_out.push_back(items[i].code);
        const size_t base = src_out.size();
        src_out.resize(base + kBN, -1);
        while (j < items.size() && items[j].code == items[i].code && items[j].occ == items[i].occ) {
          for (int q = 0; q < dc; ++q) src_out[base + items[j].slot * dc + q] = items[j].src * dc + q;
          ++j;
        }
        i = j;
      }
    }
  };
  std::vector<std::thread> pool;
  for (unsigned w = 1; w < nth; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto& th : pool) th.join();
  for (auto& cc : part_count)
    for (int c = 0; c < kNumCodes; ++c) plan.code_count[c] += cc[c];
  for (int c = 0; c < kNumCodes; ++c) plan.n_pairs += plan.code_count[c];
  // 6. concatenate
  plan.tile_off.resize(n_tiles + 1);
  int64_t e = 0;
  for (int64_t tile = 0; tile < n_tiles; ++tile) {
    plan.tile_off[tile] = int(e);
    e += int64_t(t_code[tile].size());
  }
  if (e > INT32_MAX) throw PlanError(1, "plan too large for int32 entry offsets");
  plan.tile_off[n_tiles] = int(e);
  plan.entry_code.resize(e);
  plan.entry_src.resize(size_t(e) * kBN);
  {  // parallel over tile ranges (the copy of a level-7 plan is ~1.5 GB)
    auto cwork = [&](unsigned w) {
      for (int64_t tile = int64_t(w) * n_tiles / nth; tile < int64_t(w + 1) * n_tiles / nth; ++tile) {
        std::copy(t_code[tile].begin(), t_code[tile].end(), plan.entry_code.begin() + plan.tile_off[tile]);
        std::copy(t_src[tile].begin(), t_src[tile].end(),
                  plan.entry_src.begin() + size_t(plan.tile_off[tile]) * kBN);
        std::vector<int>().swap(t_src[tile]);
      }
    };
    std::vector<std::thread> cp;
    for (unsigned w = 1; w < nth; ++w) cp.emplace_back(cwork, w);
    cwork(0);
    for (auto& th : cp) th.join();
  }
  return plan;
}

// Pair-mode plan (sparse trees): entries are runs of up to BN/dc pairs that
// share one transfer vector, whatever their targets; `entries_per_tile`
// consecutive entries form a tile (one CTA).  Entry e, slot s produces result
// row e*(BN/dc)+s; red_* is the per-target CSR of those rows (rows ascending)
// for the ordered reduction.
struct PairReduce {
  std::vector<int64_t> tgt, off;
  std::vector<int> frow;
  int64_t n_frows = 0;
};

inline HostPlan build_plan_pairs(int64_t n_targets, const int64_t* tgt, const int64_t* off, const int64_t* src,
                                 const int16_t* codes, int dc, const std::array<int, kNumCodes>& opkey,
                                 int64_t n_rows, int entries_per_tile, PairReduce& red) {
  HostPlan plan;
  plan.dc = dc;
  const int tpt = kBN / dc;
  struct P {
    int key, code;
    int64_t row, src;
  };
  std::vector<P> pairs;
  for (int64_t i = 0; i < n_targets; ++i) {
    if (tgt[i] < 0 || tgt[i] >= n_rows) throw PlanError(1, "target row out of range");
    if (off[i + 1] < off[i]) throw PlanError(1, "offsets must be non-decreasing");
    for (int64_t q = off[i]; q < off[i + 1]; ++q) {
      const int c = codes[q];
      if (c < 0 || c >= kNumCodes) throw PlanError(1, "transfer vector outside [-3,3]^3");
      if (opkey[c] < 0) {
        int t0, t1, t2;
        tcode_decode(c, t0, t1, t2);
        throw PlanError(2, "no operator for transfer vector (" + std::to_string(t0) + ", " + std::to_string(t1) +
                               ", " + std::to_string(t2) + ")");
      }
      if (src[q] < 0 || src[q] >= n_rows) throw PlanError(1, "source row out of range");
      pairs.push_back({opkey[c], c, tgt[i], src[q]});
      plan.code_count[c] += 1;
    }
  }
  plan.n_pairs = int64_t(pairs.size());
  std::stable_sort(pairs.begin(), pairs.end(), [](const P& a, const P& b) {
    if (a.key != b.key) return a.key < b.key;
    if (a.code != b.code) return a.code < b.code;
    return a.row < b.row;
  });
  std::vector<std::pair<int64_t, int>> tf;  // (target row, result row)
  tf.reserve(pairs.size());
  for (size_t i = 0; i < pairs.size();) {
    size_t j = i;
    while (j < pairs.size() && pairs[j].code == pairs[i].code) ++j;
    for (size_t a = i; a < j; a += tpt) {
      const int64_t e = int64_t(plan.entry_code.size());
      plan.entry_code.push_back(pairs[i].code);
      plan.entry_src.resize(size_t(e + 1) * kBN, -1);
      for (size_t b = a; b < std::min(j, a + tpt); ++b) {
        const int sl = int(b - a);
        for (int q = 0; q < dc; ++q) plan.entry_src[size_t(e) * kBN + sl * dc + q] = int(pairs[b].src * dc + q);
        tf.emplace_back(pairs[b].row, int(e * tpt + sl));
      }
    }
    i = j;
  }
  const int64_t E = plan.n_entries();
  if (E * tpt > INT32_MAX) throw PlanError(1, "pair plan too large");
  plan.n_tiles = (E + entries_per_tile - 1) / entries_per_tile;
  plan.tile_off.resize(plan.n_tiles + 1);
  for (int64_t t = 0; t <= plan.n_tiles; ++t) plan.tile_off[t] = int(std::min<int64_t>(t * entries_per_tile, E));
  plan.tile_col.assign(size_t(plan.n_tiles) * kBN, -1);
  std::sort(tf.begin(), tf.end());
  red.n_frows = E * tpt;
  red.tgt.clear();
  red.off.assign(1, 0);
  red.frow.resize(tf.size());
  for (size_t i = 0; i < tf.size(); ++i) {
    if (i == 0 || tf[i].first != tf[i - 1].first) {
      if (i) red.off.push_back(int64_t(i));
      red.tgt.push_back(tf[i].first);
    }
    red.frow[i] = tf[i].second;
  }
  red.off.push_back(int64_t(tf.size()));
  if (tf.empty()) red.off.assign(1, 0);
  return plan;
}

// One entry per tile over a list of virtual ids: used for the shared-basis
// per-source (m2l.py:378) and per-target (m2l.py:393) transforms, where the
// "source" of output column v is row v of the input.
inline HostPlan build_identity_plan(const std::vector<int64_t>& rows, int dc) {
  HostPlan plan;
  plan.dc = dc;
  const int tpt = kBN / dc;
  const int64_t nu = int64_t(rows.size());
  plan.n_tiles = (nu + tpt - 1) / tpt;
  plan.tile_col.assign(size_t(plan.n_tiles) * kBN, -1);
  plan.tile_off.resize(plan.n_tiles + 1);
  plan.entry_code.assign(plan.n_tiles, 0);
  plan.entry_src.assign(size_t(plan.n_tiles) * kBN, -1);
  for (int64_t k = 0; k < nu; ++k) {
    const int64_t tile = k / tpt, slot = k % tpt;
    for (int q = 0; q < dc; ++q) {
      const int v = int(rows[k] * dc + q);
      plan.tile_col[size_t(tile) * kBN + slot * dc + q] = v;
      plan.entry_src[size_t(tile) * kBN + slot * dc + q] = v;
    }
  }
  for (int64_t t = 0; t <= plan.n_tiles; ++t) plan.tile_off[t] = int(t);
  return plan;
}

}  // namespace cfm
