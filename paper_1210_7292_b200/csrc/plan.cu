// Apply plans of a level: target tiles, pair entries, hybrid, two-stage low rank, the CSR plan cache.
#include "internal.hpp"

#include <functional>
#include <thread>

namespace cfm {

// ------------------------------------------------------------------ planning
std::vector<int16_t> codes_from_t(int64_t P, const int8_t* t) {
  std::vector<int16_t> codes(P);
  for (int64_t q = 0; q < P; ++q) {
    const int t0 = t[3 * q], t1 = t[3 * q + 1], t2 = t[3 * q + 2];
    if (t0 < -3 || t0 > 3 || t1 < -3 || t1 > 3 || t2 < -3 || t2 > 3) {
      throw Error(CFM_ERR_PRECOMPUTE, "no operator for transfer vector (" + std::to_string(t0) + ", " +
                                          std::to_string(t1) + ", " + std::to_string(t2) + ")");
    }
    codes[q] = int16_t(tcode(t0, t1, t2));
  }
  return codes;
}

Group& group_for_level(cfm_handler* h, int level) {
  auto it = h->levels.find(level);
  if (it == h->levels.end())
    throw Error(CFM_ERR_PRECOMPUTE, "no operators precomputed for level " + std::to_string(level));
  auto git = h->groups.find(it->second.first);
  if (git == h->groups.end()) throw Error(CFM_ERR_PRECOMPUTE, "level group has no operators");
  return git->second;
}

// Two-stage low-rank plans from a level's target-tile plan (Group::has_ts).
// Stage 1: source tiles (64 sources of one class) x ts_nb entries (one per
// 128-row block of the class stack); each entry's 128 x 64 result is written
// to the sources' Y rows (Y: n_rows x ts_ldy, columns by ts_colmap).
// Stage 2: the target tiles with every entry (t, 64 sources) split into its
// 16-wide rank segments j (operator id 2 k + j, k = transfer index); the B
// tile of an entry is gathered from the 64 sources' Y rows at column
// ts_opcol[2 k + j].  Taken only when stage 1 computes at most ~1.7x the rank rows the
// pairs need and Y fits CFM_LR_TWOSTAGE_GB (default 24 GB).
void build_two_stage_plan(const Group& g, LevelPlan& lp) {
  const HostPlan& hp = lp.hp;
  const int64_t n_rows = lp.n_rows;
  const int ntr = g.ts_ntr, nb = g.ts_nb;
  std::vector<int8_t> mn(size_t(n_rows) * 3, 127), mx(size_t(n_rows) * 3, -128);
  std::vector<char> used(n_rows, 0);
  int64_t need_rows = 0;
  const int64_t E = hp.n_entries();
  for (int64_t e = 0; e < E; ++e) {
    const int c = hp.entry_code[e];
    const int k = g.fullmap.op[c];
    if (k < 0 || k >= ntr || g.ts_rank[k] <= 0) return;
    int t[3];
    tcode_decode(c, t[0], t[1], t[2]);
    for (int col = 0; col < kBN; ++col) {
      const int v = hp.entry_src[size_t(e) * kBN + col];
      if (v < 0) continue;
      used[v] = 1;
      need_rows += g.ts_rank[k];
      for (int a = 0; a < 3; ++a) {
        mn[size_t(v) * 3 + a] = std::min<int8_t>(mn[size_t(v) * 3 + a], int8_t(t[a]));
        mx[size_t(v) * 3 + a] = std::max<int8_t>(mx[size_t(v) * 3 + a], int8_t(t[a]));
      }
    }
  }
  std::vector<int8_t> cls(n_rows, -1);
  std::vector<std::vector<int64_t>> by_cls(8);
  for (int64_t v = 0; v < n_rows; ++v) {
    if (!used[v]) continue;
    int b = 0;
    for (int a = 0; a < 3; ++a) {
      if (mx[size_t(v) * 3 + a] <= 2) continue;        // fits [-3, 2]
      if (mn[size_t(v) * 3 + a] >= -2) b |= 1 << a;     // fits [-2, 3]
      else return;                                      // not an octree far list
    }
    cls[v] = int8_t(b);
    by_cls[b].push_back(v);
  }
  // stage 1 plan
  HostPlan p1;
  for (int b = 0; b < 8; ++b)
    for (size_t i = 0; i < by_cls[b].size(); i += kBN) {
      p1.n_tiles++;
      p1.tile_off.push_back(int(p1.entry_code.size()));
      std::vector<int> cols(kBN, -1);
      for (int c = 0; c < kBN && i + c < by_cls[b].size(); ++c) cols[c] = int(by_cls[b][i + c]);
      p1.tile_col.insert(p1.tile_col.end(), cols.begin(), cols.end());
      for (int blk = 0; blk < nb; ++blk) {
        p1.entry_code.push_back(b * nb + blk);
        p1.entry_src.insert(p1.entry_src.end(), cols.begin(), cols.end());
      }
    }
  p1.tile_off.push_back(int(p1.entry_code.size()));
  static const double budget_gb = [] {
    const char* e = getenv("CFM_LR_TWOSTAGE_GB");
    return e ? atof(e) : 24.0;
  }();
  if (double(n_rows) * g.ts_ldy * 8 > budget_gb * 1e9) return;
  if (double(p1.n_tiles) * kBN * nb * 128 > 1.7 * double(need_rows)) return;  // sparse level: fused kernel
  // stage 2 plan: the target tiles, every entry split into its rank segments
  // (operator 2 k + j); B = the sources' Y rows from column ts_opcol[2 k + j]
  HostPlan p2;
  p2.n_tiles = hp.n_tiles;
  p2.tile_col = hp.tile_col;
  p2.tile_off.reserve(hp.n_tiles + 1);
  for (int64_t t = 0; t < hp.n_tiles; ++t) {
    p2.tile_off.push_back(int(p2.entry_code.size()));
    for (int e = hp.tile_off[t]; e < hp.tile_off[t + 1]; ++e) {
      const int k = g.fullmap.op[hp.entry_code[e]];
      for (int j = 0; j * 16 < g.ts_rank[k]; ++j) {
        p2.entry_code.push_back(2 * k + j);
        p2.entry_src.insert(p2.entry_src.end(), hp.entry_src.begin() + size_t(e) * kBN,
                            hp.entry_src.begin() + size_t(e + 1) * kBN);
      }
    }
  }
  p2.tile_off.push_back(int(p2.entry_code.size()));
  if (p2.n_entries() >= (int64_t(1) << 31) / kBN) return;
  lp.ts_tile_tmin.assign(p2.n_tiles, lp.n_rows);
  for (int64_t t = 0; t < p2.n_tiles; ++t)
    for (int c = 0; c < kBN; ++c) {
      const int v = p2.tile_col[size_t(t) * kBN + c];
      if (v >= 0) lp.ts_tile_tmin[t] = std::min<int64_t>(lp.ts_tile_tmin[t], v);
    }
  for (int64_t t = p2.n_tiles - 1; t > 0; --t)  // monotone: "rows below tmin[t] are final after tiles < t"
    lp.ts_tile_tmin[t - 1] = std::min(lp.ts_tile_tmin[t - 1], lp.ts_tile_tmin[t]);
  lp.ts1 = std::move(p1);
  lp.ts2 = std::move(p2);
  push_plan(lp.ts1, lp.ts1_col, lp.ts1_off, lp.ts1_code, lp.ts1_src);
  push_plan(lp.ts2, lp.ts2_col, lp.ts2_off, lp.ts2_code, lp.ts2_src);
  lp.ts = 1;
}

// Target-major two-stage plans (Group::has_tsT; LevelPlan::ts == 2) straight
// from the level's CSR lists.  Sources and targets are classed by the range
// pattern of their transfers (a cell whose transfers fit both ranges of an
// axis takes bit 0).  Stage 1: tiles of 64 sources of one class x tsT_nb
// entries (128-row blocks of the class's V stack); the epilogue writes the row
// (slot, a) of source s to Y_T at nbr[s][slot] + a, where nbr holds the element
// offset target * ldY + rho_T[class(target)][k] of the pair's rank run (-1: the
// source has no pair with that transfer, nothing is written and the
// corresponding Y_T columns keep the zeros of the one-time memset).  Stage 2:
// tiles of 64 targets of one class (ascending rows; tiles ordered by their
// smallest row), one entry per 128-column block of the class's U stack whose
// B rows are the targets' Y_T rows of that block -- a plain dense GEMM on the
// full-operator step kernel.
static bool build_two_stage_plan_T(const Group& g, LevelPlan& lp, int64_t n_targets, const int64_t* tgt,
                                   const int64_t* off, const int64_t* src, const int16_t* codes) {
  const int64_t n_rows = lp.n_rows;
  const int ntr = g.ts_ntr, nb = g.tsT_nb, nslots = g.tsT_nslots;
  const int64_t ldy = int64_t(nb) * 128;
  if (n_rows <= 0 || double(n_rows) * double(ldy) >= 2147483647.0) return false;  // int32 offsets
  static const double budget_gb = [] {
    const char* e = getenv("CFM_LR_TWOSTAGE_GB");
    return e ? atof(e) : 24.0;
  }();
  if (double(n_rows) * double(ldy) * 8 > budget_gb * 1e9) return false;
  // decoded transfer components of every code
  std::array<int8_t, 3 * kNumCodes> tc{};
  for (int c = 0; c < kNumCodes; ++c) {
    int t0, t1, t2;
    tcode_decode(c, t0, t1, t2);
    tc[3 * c] = int8_t(t0), tc[3 * c + 1] = int8_t(t1), tc[3 * c + 2] = int8_t(t2);
  }
  // pass over the pairs on host threads (46 M pairs at config 2's level 6): per target the range of
  // its transfers, per source the same through per-thread arrays merged afterwards
  std::vector<int8_t> smn(size_t(n_rows) * 3, 127), smx(size_t(n_rows) * 3, -128);
  std::vector<int8_t> tcls(n_targets, -1);
  int64_t need_rows = 0;
  const int nth = int(std::max<int64_t>(1, std::min<int64_t>(std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency())),
                                                               n_targets / 4096)));
  {
    std::vector<std::vector<int8_t>> tmn(nth), tmx(nth);
    std::vector<int64_t> tneed(nth, 0);
    std::vector<char> bad(nth, 0);
    auto work = [&](int w) {
      std::vector<int8_t>& lmn = tmn[w];
      std::vector<int8_t>& lmx = tmx[w];
      lmn.assign(size_t(n_rows) * 3, 127);
      lmx.assign(size_t(n_rows) * 3, -128);
      for (int64_t i = n_targets * w / nth; i < n_targets * (w + 1) / nth; ++i) {
        if (tgt[i] < 0 || tgt[i] >= n_rows) { bad[w] = 1; return; }
        int8_t mn[3] = {127, 127, 127}, mx[3] = {-128, -128, -128};
        for (int64_t q = off[i]; q < off[i + 1]; ++q) {
          const int c = codes[q];
          const int k = (c >= 0 && c < kNumCodes) ? g.fullmap.op[c] : -1;
          if (k < 0 || k >= ntr || g.ts_rank[k] <= 0) { bad[w] = 1; return; }
          tneed[w] += g.ts_rank[k];
          const int64_t v = src[q];
          if (v < 0 || v >= n_rows) { bad[w] = 1; return; }
          for (int a = 0; a < 3; ++a) {
            const int8_t t = tc[3 * c + a];
            mn[a] = std::min(mn[a], t), mx[a] = std::max(mx[a], t);
            lmn[size_t(v) * 3 + a] = std::min(lmn[size_t(v) * 3 + a], t);
            lmx[size_t(v) * 3 + a] = std::max(lmx[size_t(v) * 3 + a], t);
          }
        }
        if (off[i + 1] == off[i]) continue;
        int b = 0;
        for (int a = 0; a < 3; ++a) {
          if (mx[a] <= 2 && mn[a] >= -3) continue;
          if (mn[a] >= -2 && mx[a] <= 3) b |= 1 << a;
          else { bad[w] = 1; return; }  // not an octree far list
        }
        tcls[i] = int8_t(b);
      }
    };
    std::vector<std::thread> th;
    for (int w = 1; w < nth; ++w) th.emplace_back(work, w);
    work(0);
    for (auto& t : th) t.join();
    for (int w = 0; w < nth; ++w) {
      if (bad[w]) return false;
      need_rows += tneed[w];
      for (size_t j = 0; j < smn.size(); ++j) {
        smn[j] = std::min(smn[j], tmn[w][j]);
        smx[j] = std::max(smx[j], tmx[w][j]);
      }
    }
  }
  std::vector<int8_t> scls(n_rows, -1);
  std::vector<std::vector<int>> src_by(8);
  for (int64_t v = 0; v < n_rows; ++v) {
    if (smx[size_t(v) * 3] == -128) continue;
    int b = 0;
    for (int a = 0; a < 3; ++a) {
      if (smx[size_t(v) * 3 + a] <= 2 && smn[size_t(v) * 3 + a] >= -3) continue;
      if (smn[size_t(v) * 3 + a] >= -2 && smx[size_t(v) * 3 + a] <= 3) b |= 1 << a;
      else return false;
    }
    scls[v] = int8_t(b);
    src_by[b].push_back(int(v));
  }
  int64_t tiles1 = 0;
  for (int b = 0; b < 8; ++b) tiles1 += (int64_t(src_by[b].size()) + kBN - 1) / kBN;
  if (double(tiles1) * kBN * nb * 128 > 1.7 * double(need_rows)) return false;  // sparse level: fused kernel
  // per (source, class slot): where the pair's rank run lands in Y_T
  std::vector<int> nbr(size_t(n_rows) * nslots, -1);
  {
    std::vector<char> tseen(n_rows, 0);
    for (int64_t i = 0; i < n_targets; ++i) {
      if (off[i + 1] == off[i]) continue;
      if (tseen[tgt[i]]) return false;  // a target listed twice: its Y_T row would be shared
      tseen[tgt[i]] = 1;
    }
    // (a (source, class slot) belongs to one pair of an octree list; a second pair on the same
    // entry is not an octree list and refuses the plan)
    std::vector<char> bad(nth, 0);
    auto work = [&](int w) {
      for (int64_t i = n_targets * w / nth; i < n_targets * (w + 1) / nth; ++i) {
        if (off[i + 1] == off[i]) continue;
        const int ct = tcls[i];
        for (int64_t q = off[i]; q < off[i + 1]; ++q) {
          const int k = g.fullmap.op[codes[q]];
          const int64_t v = src[q];
          const int slot = g.tsT_slot[size_t(scls[v]) * ntr + k];
          const int rho = g.tsT_rho[size_t(ct) * ntr + k];
          if (slot < 0 || rho < 0) { bad[w] = 1; return; }
          int expected = -1;  // (compare-exchange: a duplicate is caught also when two threads race for it)
          if (!__atomic_compare_exchange_n(&nbr[size_t(v) * nslots + slot], &expected, int(tgt[i] * ldy + rho), false,
                                           __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
            bad[w] = 1;
            return;
          }
        }
      }
    };
    std::vector<std::thread> th;
    for (int w = 1; w < nth; ++w) th.emplace_back(work, w);
    work(0);
    for (auto& t : th) t.join();
    for (int w = 0; w < nth; ++w)
      if (bad[w]) return false;
  }
  // stage 1 plan: tiles of 64 same-class sources (ascending rows), ordered by their
  // first row, so a host-buffer apply can start on the first multipole slabs
  struct T1 { int cls; int first; int count; int minrow; };
  std::vector<T1> t1;
  for (int b = 0; b < 8; ++b)
    for (size_t i = 0; i < src_by[b].size(); i += kBN)
      t1.push_back({b, int(i), int(std::min<size_t>(kBN, src_by[b].size() - i)), src_by[b][i]});
  std::stable_sort(t1.begin(), t1.end(), [](const T1& a, const T1& b) { return a.minrow < b.minrow; });
  HostPlan p1;
  lp.ts1_need.assign(t1.size(), 0);
  for (size_t t = 0; t < t1.size(); ++t) {
    p1.n_tiles++;
    p1.tile_off.push_back(int(p1.entry_code.size()));
    std::vector<int> cols(kBN, -1);
    for (int c = 0; c < t1[t].count; ++c) cols[c] = src_by[t1[t].cls][t1[t].first + c];
    p1.tile_col.insert(p1.tile_col.end(), cols.begin(), cols.end());
    lp.ts1_need[t] = std::max<int64_t>(t ? lp.ts1_need[t - 1] : 0, cols[t1[t].count - 1]);
    for (int blk = 0; blk < g.tsT_nblk[t1[t].cls]; ++blk) {
      p1.entry_code.push_back(t1[t].cls * nb + blk);
      p1.entry_src.insert(p1.entry_src.end(), cols.begin(), cols.end());
    }
  }
  p1.tile_off.push_back(int(p1.entry_code.size()));
  // stage 2 plan: tiles of one class, ordered by their smallest target row
  std::vector<std::vector<int>> tgt_by(8);
  for (int64_t i = 0; i < n_targets; ++i)
    if (tcls[i] >= 0) tgt_by[tcls[i]].push_back(int(tgt[i]));
  struct T2 { int cls; int first; int count; int minrow; };
  std::vector<T2> t2;
  for (int b = 0; b < 8; ++b) {
    std::sort(tgt_by[b].begin(), tgt_by[b].end());
    for (size_t i = 0; i < tgt_by[b].size(); i += kBN)
      t2.push_back({b, int(i), int(std::min<size_t>(kBN, tgt_by[b].size() - i)), tgt_by[b][i]});
  }
  std::stable_sort(t2.begin(), t2.end(), [](const T2& a, const T2& b) { return a.minrow < b.minrow; });
  HostPlan p2;
  p2.n_tiles = int64_t(t2.size());
  lp.ts_tile_tmin.assign(t2.size(), n_rows);
  lp.ts2_need.assign(t2.size(), 0);
  for (size_t t = 0; t < t2.size(); ++t) {
    p2.tile_off.push_back(int(p2.entry_code.size()));
    std::vector<int> cols(kBN, -1);
    for (int c = 0; c < t2[t].count; ++c) cols[c] = tgt_by[t2[t].cls][t2[t].first + c];
    p2.tile_col.insert(p2.tile_col.end(), cols.begin(), cols.end());
    lp.ts_tile_tmin[t] = t2[t].minrow;
    lp.ts2_need[t] = std::max<int64_t>(t ? lp.ts2_need[t - 1] : 0, cols[t2[t].count - 1]);
    for (int blk = 0; blk < g.tsT_nblk[t2[t].cls]; ++blk) {
      p2.entry_code.push_back(t2[t].cls * nb + blk);
      for (int c = 0; c < kBN; ++c) p2.entry_src.push_back(cols[c] >= 0 ? cols[c] * nb + blk : -1);
    }
  }
  p2.tile_off.push_back(int(p2.entry_code.size()));
  for (int64_t t = p2.n_tiles - 1; t > 0; --t)
    lp.ts_tile_tmin[t - 1] = std::min(lp.ts_tile_tmin[t - 1], lp.ts_tile_tmin[t]);
  lp.ts1 = std::move(p1);
  lp.ts2 = std::move(p2);
  push_plan(lp.ts1, lp.ts1_col, lp.ts1_off, lp.ts1_code, lp.ts1_src);
  push_plan(lp.ts2, lp.ts2_col, lp.ts2_off, lp.ts2_code, lp.ts2_src);
  upload(lp.tsT_nbr, nbr);
  lp.ts = 2;
  return true;
}

// Hybrid plans (CFM_HYBRID=0 disables): measured at config 2 the step kernel
// drops 50.56 -> 50.28 ms; with all reductions of a step in one launch the
// step goes 50.60 -> 50.41 ms.  Read at every plan build; a forced
// CFM_PLAN_MODE disables it.
bool use_hybrid() {
  const char* e = getenv("CFM_HYBRID");
  return (!e || atoi(e) != 0) && !getenv("CFM_PLAN_MODE");
}

// Upload a pair-mode plan's device arrays (entries, reduction, filled columns).
void push_pair_plan(LevelPlan& lp) {
  push_plan(lp.hp, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src);
  upload(lp.r_tgt, lp.red.tgt);
  upload(lp.r_off, lp.red.off);
  upload(lp.r_frow, lp.red.frow);
  const int64_t E = lp.hp.n_entries();
  std::vector<unsigned char> nc(std::max<int64_t>(E, 1), 0);
  for (int64_t e = 0; e < E; ++e)
    for (int c = kBN - 1; c >= 0; --c)
      if (lp.hp.entry_src[size_t(e) * kBN + c] >= 0) {
        nc[e] = static_cast<unsigned char>(c + 1);
        break;
      }
  upload(lp.entry_ncols, nc);
}

// Hybrid split of a dense full-operator target-tile plan (LevelPlan::hyb).
void build_hybrid_plan(cfm_handler* h, LevelPlan& lp, int64_t n_targets, const int64_t* tgt,
                              const int64_t* off, const int64_t* src, const int16_t* codes,
                              const std::array<int, kNumCodes>& key) {
  const HostPlan& hp = lp.hp;
  std::vector<char> leftover_tile(hp.n_tiles, 0);
  std::vector<char> leftover_row(lp.n_rows, 0);
  {  // tiles less than half full (parallel scan of the entries)
    const unsigned nth = unsigned(std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()),
                                                    std::max<int64_t>(1, hp.n_tiles / 256)));
    auto scan = [&](unsigned w) {
      for (int64_t t = int64_t(w) * hp.n_tiles / nth; t < int64_t(w + 1) * hp.n_tiles / nth; ++t) {
        int64_t valid = 0;
        const int64_t slots = int64_t(hp.tile_off[t + 1] - hp.tile_off[t]) * kBN;
        for (size_t i = size_t(hp.tile_off[t]) * kBN; i < size_t(hp.tile_off[t + 1]) * kBN; ++i)
          valid += hp.entry_src[i] >= 0;
        leftover_tile[t] = slots != 0 && 2 * valid < slots;
      }
    };
    std::vector<std::thread> th;
    for (unsigned w = 1; w < nth; ++w) th.emplace_back(scan, w);
    scan(0);
    for (auto& x : th) x.join();
  }
  int64_t n_left = 0;
  for (int64_t t = 0; t < hp.n_tiles; ++t) {
    if (!leftover_tile[t]) continue;
    ++n_left;
    for (int c = 0; c < kBN; ++c) {
      const int v = hp.tile_col[size_t(t) * kBN + c];
      if (v >= 0) leftover_row[v] = 1;
    }
  }
  if (n_left == 0 || n_left == hp.n_tiles) return;
  auto hy = std::make_shared<HybridPlan>();
  HostPlan& mn = hy->main;
  mn.bn = hp.bn;
  mn.dc = hp.dc;
  // kept tiles longest first (row order kept among equally long tiles): the
  // shorter boundary-class tiles run last and fill the launch's tail (this
  // plan only serves device-resident applies, which need no row order)
  std::vector<int64_t> kept;
  for (int64_t t = 0; t < hp.n_tiles; ++t)
    if (!leftover_tile[t]) kept.push_back(t);
  std::stable_sort(kept.begin(), kept.end(), [&](int64_t a, int64_t b) {
    return hp.tile_off[a + 1] - hp.tile_off[a] > hp.tile_off[b + 1] - hp.tile_off[b];
  });
  const int max_e = kept.empty() ? 0 : hp.tile_off[kept[0] + 1] - hp.tile_off[kept[0]];
  for (int64_t t : kept) hy->n_long += (hp.tile_off[t + 1] - hp.tile_off[t]) * 10 >= max_e * 9;
  {  // copy the kept tiles (offsets first, then the entries in parallel)
    mn.n_tiles = int64_t(kept.size());
    mn.tile_off.resize(kept.size() + 1);
    mn.tile_col.resize(kept.size() * kBN);
    int64_t ne = 0;
    for (size_t i = 0; i < kept.size(); ++i) {
      mn.tile_off[i] = int(ne);
      ne += hp.tile_off[kept[i] + 1] - hp.tile_off[kept[i]];
    }
    mn.tile_off[kept.size()] = int(ne);
    mn.entry_code.resize(ne);
    mn.entry_src.resize(size_t(ne) * kBN);
    const unsigned nth = unsigned(std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()),
                                                    std::max<int64_t>(1, int64_t(kept.size()) / 256)));
    auto copy = [&](unsigned w) {
      for (size_t i = kept.size() * w / nth; i < kept.size() * (w + 1) / nth; ++i) {
        const int64_t t = kept[i];
        std::copy(hp.tile_col.begin() + t * kBN, hp.tile_col.begin() + (t + 1) * kBN, mn.tile_col.begin() + i * kBN);
        std::copy(hp.entry_code.begin() + hp.tile_off[t], hp.entry_code.begin() + hp.tile_off[t + 1],
                  mn.entry_code.begin() + mn.tile_off[i]);
        std::copy(hp.entry_src.begin() + size_t(hp.tile_off[t]) * kBN, hp.entry_src.begin() + size_t(hp.tile_off[t + 1]) * kBN,
                  mn.entry_src.begin() + size_t(mn.tile_off[i]) * kBN);
      }
    };
    std::vector<std::thread> th;
    for (unsigned w = 1; w < nth; ++w) th.emplace_back(copy, w);
    copy(0);
    for (auto& x : th) x.join();
  }
  // leftover targets' far lists (CSR order kept) -> pair entries
  std::vector<int64_t> t2, o2{0}, s2;
  std::vector<int16_t> c2;
  for (int64_t i = 0; i < n_targets; ++i) {
    if (off[i + 1] <= off[i] || !leftover_row[tgt[i]]) continue;
    t2.push_back(tgt[i]);
    for (int64_t q = off[i]; q < off[i + 1]; ++q) {
      s2.push_back(src[q]);
      c2.push_back(codes[q]);
    }
    o2.push_back(int64_t(s2.size()));
  }
  LevelPlan& ax = hy->aux;
  const int nkp = round_up(h->n * h->f, kKC);
  const int64_t e_est = int64_t(s2.size()) / kBN + 1;
  int ept = std::max(1, std::min(16, int(2.5e7 / (2.0 * 128 * kBN * nkp))));
  ept = std::min<int>(ept, int(std::max<int64_t>(1, e_est / (2 * 148))));
  ax.hp = build_plan_pairs(int64_t(t2.size()), t2.data(), o2.data(), s2.data(), c2.data(), 1, key, lp.n_rows, ept,
                           ax.red);
  ax.mode = 1;
  ax.dc = 1;
  ax.n_rows = lp.n_rows;
  push_pair_plan(ax);
  static uint64_t hyb_gen = uint64_t(1) << 62;
  ax.gen = ++hyb_gen;
  push_plan(mn, hy->tile_col, hy->tile_off, hy->entry_code, hy->entry_src);
  lp.hyb = std::move(hy);
}

uint64_t next_plan_gen() {
  static std::atomic<uint64_t> plan_gen{0};
  return ++plan_gen;
}

// Host<->device copy pipeline of a target-tile level: row slabs, and per tile
// the multipole / locals slabs it needs (tile_rows(t, min target row, max
// target row, max source row)); every CTA (tile x row block) writing a slab is
// counted so the download of a finished slab can start while the kernel runs.
void set_slab_plan(cfm_handler* h, int level, LevelPlan& lp,
                   const std::function<void(int64_t, int64_t&, int64_t&, int64_t&)>& tile_rows) {
  const int64_t n_rows = lp.n_rows;
  const int64_t nt = lp.hp.n_tiles;
  // slabs of ~32K rows (at most 16); CFM_SLAB_ROWS / CFM_MAX_SLABS for experiments
  static const int64_t slab_rows = [] {
    const char* e = getenv("CFM_SLAB_ROWS");
    return e ? std::max<int64_t>(1024, atoll(e)) : int64_t(32768);
  }();
  static const int64_t max_slabs = [] {
    const char* e = getenv("CFM_MAX_SLABS");
    return e ? std::max<int64_t>(2, atoll(e)) : int64_t(16);
  }();
  const char* min_rows_e = getenv("CFM_PIPE_MIN_ROWS");  // levels with fewer rows are not host-pipelined
  const int64_t min_rows = min_rows_e ? atoll(min_rows_e) : int64_t(0);  // (read per plan: a test pipelines small levels)
  int S = int(std::min<int64_t>(max_slabs, std::max<int64_t>(1, n_rows / slab_rows)));
  if (min_rows > 0) S = n_rows >= min_rows ? std::max(S, 2) : 1;
  // the last slab's download cannot start before the kernel's last wave
  // ends: split it into halves, quarters, eighths (CFM_SLAB_TAIL=0: uniform)
  static const int slab_tail = [] {
    const char* e = getenv("CFM_SLAB_TAIL");
    return e ? std::max(0, atoi(e)) : 3;
  }();
  lp.slab_row0.clear();
  for (int k = 0; k < S; ++k) lp.slab_row0.push_back(n_rows * k / S);
  if (S >= 2) {
    const int64_t a = n_rows * (S - 1) / S, len = n_rows - a;
    int64_t r = a;
    for (int d = 1; d <= slab_tail && S + d <= 16 && (len >> d) >= 1024; ++d) {
      r += len >> d;
      lp.slab_row0.push_back(r);
    }
  }
  lp.slab_row0.push_back(n_rows);
  const int S_all = int(lp.slab_row0.size()) - 1;
  lp.n_slabs = S_all;
  auto slab_of = [&](int64_t row) {
    const auto it = std::upper_bound(lp.slab_row0.begin(), lp.slab_row0.end(), row);
    return int(std::min<int64_t>(S_all - 1, std::max<int64_t>(0, (it - lp.slab_row0.begin()) - 1)));
  };
  std::vector<int> need_mp(nt, 0), need_loc(nt, 0), lo(nt, 0), hi(nt, -1);
  lp.slab_expected.assign(S_all, 0);
  const int nrb = (group_for_level(h, level).dense.rows + 127) / 128;
  for (int64_t t = 0; t < nt; ++t) {
    int64_t tmin, tmax, smax;
    tile_rows(t, tmin, tmax, smax);  // slab_of is monotonic: the extreme rows give the extreme slabs
    int l = S_all, hh = -1, m = 0;
    if (tmax >= 0) l = slab_of(tmin), hh = slab_of(tmax);
    if (smax >= 0) m = slab_of(smax) + 1;
    if (hh < 0) { l = 0; hh = -1; }
    need_mp[t] = m;
    need_loc[t] = hh + 1;
    lo[t] = l;
    hi[t] = hh;
    for (int k = l; k <= hh; ++k) lp.slab_expected[k] += unsigned(nrb);
  }
  upload(lp.p_need_mp, need_mp);
  upload(lp.p_need_loc, need_loc);
  upload(lp.p_lo, lo);
  upload(lp.p_hi, hi);
}

LevelPlan build_level_plan(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt,
                                  const int64_t* off, const int64_t* src, const int16_t* codes, int data_complex,
                                  int64_t n_rows) {
  Group& g = group_for_level(h, level);
  const int dc = (data_complex && !h->op_complex) ? 2 : 1;
  if (h->op_complex && !data_complex)
    throw Error(CFM_ERR_VALUE, "complex operators need complex128 expansions (engine.py:99)");
  std::array<int, kNumCodes> key;
  for (int c = 0; c < kNumCodes; ++c) key[c] = g.valid[c] ? std::max(g.main.op[c], 0) + 1 : -1;
  if (g.kind == kShared)
    for (int c = 0; c < kNumCodes; ++c) key[c] = g.valid[c] ? c : -1;
  LevelPlan lp;
  try {
    const double tp0 = trace_on() ? wall_ms() : 0.0;
    lp.hp = build_plan_csr(n_targets, tgt, off, src, codes, dc, key, n_rows);
    if (trace_on()) fprintf(stderr, "[cfm plan L%d] build_plan_csr %.1f ms (%lld pairs)\n", level, wall_ms() - tp0,
                            (long long)(n_targets ? off[n_targets] : 0));
    const double slots = double(lp.hp.n_entries()) * kBN;
    lp.target_fill = slots > 0 ? double(lp.hp.n_pairs) * dc / slots : 1.0;
    const char* m = getenv("CFM_PLAN_MODE");
    const bool force_pair = m && !strcmp(m, "pair");
    const bool force_target = m && !strcmp(m, "target");
    if (force_pair || (!force_target && lp.target_fill < 0.6)) {
      // dense: ~25 MFLOP of row-block work per CTA (l = 9: 2 entries, l = 5: 11) so
      // sparse levels still give many waves of CTAs and a short tail
      const int nkp = round_up(h->n * h->f, kKC);
      static const int ept_env = [] {
        const char* e = getenv("CFM_PAIR_EPT");
        return e ? atoi(e) : 0;
      }();
      // ... and at least ~2 CTAs per SM where the level has the entries for it
      // (a small level in few long CTAs is latency-bound)
      const int64_t e_est = lp.hp.n_pairs * dc / kBN + 1;
      const int ept_occ = int(std::max<int64_t>(1, e_est / (2 * 148)));
      int ept = g.kind == kDense ? std::max(1, std::min(16, int(2.5e7 / (2.0 * 128 * kBN * nkp)))) : 16;
      ept = std::min(ept, ept_occ);
      if (ept_env > 0) ept = ept_env;
      lp.hp = build_plan_pairs(n_targets, tgt, off, src, codes, dc, key, n_rows, ept, lp.red);
      lp.mode = 1;
      upload(lp.r_tgt, lp.red.tgt);
      upload(lp.r_off, lp.red.off);
      upload(lp.r_frow, lp.red.frow);
    }
  } catch (const PlanError& e) {
    throw Error(e.code == 2 ? CFM_ERR_PRECOMPUTE : CFM_ERR_VALUE, e.what());
  }
  const double tu0 = trace_on() ? wall_ms() : 0.0;
  lp.dc = dc;
  lp.n_rows = n_rows;
  {  // row spans a host-buffer apply moves (engine.py's thread chunks are contiguous target ranges)
    int64_t slo = n_rows, shi = 0, tlo = n_rows, thi = 0;
    const int64_t P = n_targets ? off[n_targets] : 0;
    for (int64_t i = 0; i < n_targets; ++i)
      if (off[i + 1] > off[i]) tlo = std::min(tlo, tgt[i]), thi = std::max(thi, tgt[i] + 1);
    for (int64_t q = 0; q < P; ++q) slo = std::min(slo, src[q]), shi = std::max(shi, src[q] + 1);
    lp.src_lo = std::min(slo, shi), lp.src_hi = shi, lp.tgt_lo = std::min(tlo, thi), lp.tgt_hi = thi;
  }
  if (lp.mode != 0 || lp.hp.n_tiles == 0)  // (target tiles are uploaded after their re-ordering below)
    push_plan(lp.hp, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src);
  const int64_t E = lp.hp.n_entries();
  if (lp.mode == 1) {
    // filled columns per pair entry (slots are filled from column 0): the
    // full-operator kernel skips the empty trailing 8-column tiles
    std::vector<unsigned char> nc(std::max<int64_t>(E, 1), 0);
    for (int64_t e = 0; e < E; ++e)
      for (int c = kBN - 1; c >= 0; --c)
        if (lp.hp.entry_src[size_t(e) * kBN + c] >= 0) {
          nc[e] = static_cast<unsigned char>(c + 1);
          break;
        }
    upload(lp.entry_ncols, nc);
  }
  // distinct targets / sources (SA transforms and accounting)
  {
    std::vector<char> seen_t(n_rows, 0), seen_s(n_rows, 0);
    for (int64_t i = 0; i < n_targets; ++i)
      if (off[i + 1] > off[i]) {
        seen_t[tgt[i]] = 1;
        for (int64_t q = off[i]; q < off[i + 1]; ++q) seen_s[src[q]] = 1;
      }
    for (int64_t r = 0; r < n_rows; ++r) {
      if (seen_t[r]) lp.targets.push_back(r);
      if (seen_s[r]) lp.sources.push_back(r);
    }
  }
  if (g.kind == kShared) {
    lp.src_plan = build_identity_plan(lp.sources, dc);
    lp.tgt_plan = build_identity_plan(lp.targets, dc);
    push_plan(lp.src_plan, lp.s_tile_col, lp.s_tile_off, lp.s_entry_code, lp.s_entry_src);
    push_plan(lp.tgt_plan, lp.t_tile_col, lp.t_tile_off, lp.t_entry_code, lp.t_entry_src);
  }
  if (lp.mode == 0 && lp.hp.n_tiles > 0) {
    // dispatch order ~ row order (tiles stay class-pure; a target's entry order
    // is unchanged, so results are bitwise identical), which lets the host
    // copies of multipoles/locals run in row slabs alongside the kernel
    HostPlan& hp = lp.hp;
    const int64_t nt = hp.n_tiles;
    std::vector<int64_t> tmin(nt, INT64_MAX);
    for (int64_t t = 0; t < nt; ++t)
      for (int c = 0; c < kBN; ++c) {
        const int v = hp.tile_col[size_t(t) * kBN + c];
        if (v >= 0) tmin[t] = std::min<int64_t>(tmin[t], v / dc);
      }
    std::vector<int64_t> ord(nt);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return tmin[a] < tmin[b]; });
    HostPlan np_;
    np_.bn = hp.bn; np_.dc = hp.dc; np_.n_tiles = nt; np_.n_pairs = hp.n_pairs; np_.code_count = hp.code_count;
    np_.tile_col.resize(hp.tile_col.size());
    np_.tile_off.resize(nt + 1);
    np_.entry_code.reserve(hp.entry_code.size());
    np_.entry_src.reserve(hp.entry_src.size());
    for (int64_t k = 0; k < nt; ++k) {
      const int64_t t = ord[k];
      std::copy(hp.tile_col.begin() + t * kBN, hp.tile_col.begin() + (t + 1) * kBN, np_.tile_col.begin() + k * kBN);
      np_.tile_off[k] = int(np_.entry_code.size());
      for (int e = hp.tile_off[t]; e < hp.tile_off[t + 1]; ++e) {
        np_.entry_code.push_back(hp.entry_code[e]);
        np_.entry_src.insert(np_.entry_src.end(), hp.entry_src.begin() + size_t(e) * kBN,
                             hp.entry_src.begin() + size_t(e + 1) * kBN);
      }
    }
    np_.tile_off[nt] = int(np_.entry_code.size());
    lp.hp = std::move(np_);
    // a low-rank level that takes the target-major two-stage path never runs the tile plan
    // itself: no device copy of it, no two-pass slots (0.6 GB of uploads at config 2's level 6)
    if (g.kind == kLowRank && dc == 1 && g.has_tsT && two_stage_mode() >= 2)
      build_two_stage_plan_T(g, lp, n_targets, tgt, off, src, codes);
    if (lp.ts != 2) push_plan(lp.hp, lp.tile_col, lp.tile_off, lp.entry_code, lp.entry_src);
    set_slab_plan(h, level, lp, [&](int64_t t, int64_t& tmin, int64_t& tmax, int64_t& smax) {
      tmin = INT64_MAX, tmax = -1, smax = -1;
      for (int c = 0; c < kBN; ++c) {
        const int v = lp.hp.tile_col[size_t(t) * kBN + c];
        if (v >= 0) tmin = std::min<int64_t>(tmin, v / dc), tmax = std::max<int64_t>(tmax, v / dc);
      }
      for (int e = lp.hp.tile_off[t]; e < lp.hp.tile_off[t + 1]; ++e)
        for (int c = 0; c < kBN; ++c) {
          const int v = lp.hp.entry_src[size_t(e) * kBN + c];
          if (v >= 0) smax = std::max<int64_t>(smax, v / dc);
        }
    });
  }
  // per-entry slots and pass-1 runs of the two-pass paths -- built from the FINAL entry order (target-mode
  // tiles were just re-ordered by row; building them before that dropped live columns on levels whose
  // tile order changes, e.g. sphere levels forced to target tiles)
  if ((g.kind == kLowRank && lp.ts != 2) || (g.kind == kShared && g.any_fac_core)) {
    const int64_t E = lp.hp.n_entries();
    std::vector<int> slots(size_t(E) * kBN), iota(E + 1);
    for (int64_t e = 0; e < E; ++e)
      for (int c = 0; c < kBN; ++c)
        slots[size_t(e) * kBN + c] = lp.hp.entry_src[size_t(e) * kBN + c] >= 0 ? int(e * kBN + c) : -1;
    std::iota(iota.begin(), iota.end(), 0);
    upload(lp.slot_ids, slots);
    upload(lp.iota, iota);
    // runs of <= kPass1Run entries that never cross a tile boundary, so a tile
    // range [t0, t1) maps to the run range [run_start[t0], run_start[t1])
    std::vector<int> runs;
    lp.run_start.assign(lp.hp.n_tiles + 1, 0);
    for (int64_t t = 0; t < lp.hp.n_tiles; ++t) {
      lp.run_start[t] = int64_t(runs.size());
      for (int e = lp.hp.tile_off[t]; e < lp.hp.tile_off[t + 1]; e += kPass1Run) runs.push_back(e);
    }
    lp.run_start[lp.hp.n_tiles] = int64_t(runs.size());
    runs.push_back(int(E));
    lp.n_runs = int64_t(runs.size()) - 1;
    upload(lp.runs, runs);
  }
  if (g.kind == kLowRank && lp.mode == 0 && dc == 1 && lp.hp.n_tiles > 0 && lp.ts != 2 && g.has_ts)
    build_two_stage_plan(g, lp);
  if (use_hybrid() && full_mode(g, lp) && lp.mode == 0 && lp.hp.n_tiles > 0) {
    try {
      build_hybrid_plan(h, lp, n_targets, tgt, off, src, codes, key);
    } catch (const PlanError& e) {
      throw Error(e.code == 2 ? CFM_ERR_PRECOMPUTE : CFM_ERR_VALUE, e.what());
    }
  }
  if (trace_on()) fprintf(stderr, "[cfm plan L%d] uploads + hybrid / two-stage plans %.1f ms\n", level, wall_ms() - tu0);
  lp.gen = next_plan_gen();
  return lp;
}

// The level's cached plan (plan_level_* / plan_level_csr; apply_planned and
// apply_levels run it).  Ad-hoc batches of cfm_apply_level_csr never land here
// (they use the CSR plan cache below), so a cached plan is only replaced by an
// explicit re-plan of its level.
LevelPlan& make_plan(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt, const int64_t* off,
                            const int64_t* src, const int16_t* codes, int data_complex, int64_t n_rows) {
  LevelPlan lp = build_level_plan(h, level, n_targets, tgt, off, src, codes, data_complex, n_rows);
  h->plans[level] = std::move(lp);
  return h->plans[level];
}

// Plans of the reference call path (apply_level with a batch, engine.py:140-157):
// FmmPlan rebuilds the same batches on every run (engine.py:98-120), so a plan is
// cached under its exact CSR content (targets, offsets, sources, transfer vectors,
// row count, data kind) and reused when the same batch comes back.  Keys are
// compared in full (memcmp), never by hash alone.
static constexpr size_t kCsrCacheMaxEntries = 64;
static constexpr size_t kCsrCacheMaxBytes = size_t(8) << 30;

// memcmp on several threads (a config-2 batch key is ~0.6 GB)
static bool equal_mt(const void* a, const void* b, size_t bytes) {
  if (bytes < (size_t(16) << 20)) return std::memcmp(a, b, bytes) == 0;
  const int T = int(std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
  std::vector<std::thread> th;
  std::atomic<bool> eq{true};
  const size_t part = (bytes + T - 1) / T;
  for (int w = 0; w < T; ++w)
    th.emplace_back([&, w] {
      const size_t o = size_t(w) * part;
      if (o < bytes && std::memcmp(static_cast<const char*>(a) + o, static_cast<const char*>(b) + o,
                                   std::min(part, bytes - o)))
        eq = false;
    });
  for (auto& x : th) x.join();
  return eq;
}

LevelPlan& csr_plan(cfm_handler* h, int level, int64_t n_targets, const int64_t* tgt, const int64_t* off,
                           const int64_t* src, const int8_t* t, int data_complex, int64_t n_rows, bool* hit_out) {
  const int64_t P = n_targets ? off[n_targets] : 0;
  for (auto it = h->csr_cache.begin(); it != h->csr_cache.end(); ++it) {
    CsrPlanEntry& e = *it;
    if (e.level != level || e.dc_flag != data_complex || e.n_rows != n_rows || int64_t(e.tgt.size()) != n_targets ||
        int64_t(e.src.size()) != P)
      continue;
    if (n_targets && std::memcmp(e.tgt.data(), tgt, size_t(n_targets) * 8)) continue;
    if (std::memcmp(e.off.data(), off, size_t(n_targets + 1) * 8)) continue;
    if (!equal_mt(e.src.data(), src, size_t(P) * 8)) continue;
    if (!equal_mt(e.t.data(), t, size_t(P) * 3)) continue;
    h->csr_cache.splice(h->csr_cache.begin(), h->csr_cache, it);  // most recently used first
    if (hit_out) *hit_out = true;
    return h->csr_cache.front().plan;
  }
  if (hit_out) *hit_out = false;
  auto codes = codes_from_t(P, t);
  CsrPlanEntry e;
  e.plan = build_level_plan(h, level, n_targets, tgt, off, src, codes.data(), data_complex, n_rows);
  e.level = level;
  e.dc_flag = data_complex;
  e.n_rows = n_rows;
  e.tgt.assign(tgt, tgt + n_targets);
  e.off.assign(off, off + n_targets + 1);
  e.src.assign(src, src + P);
  e.t.assign(t, t + 3 * P);
  const size_t bytes = e.host_bytes();
  h->csr_cache.push_front(std::move(e));
  h->csr_cache_bytes += bytes;
  while (h->csr_cache.size() > 1 &&
         (h->csr_cache.size() > kCsrCacheMaxEntries || h->csr_cache_bytes > kCsrCacheMaxBytes)) {
    h->csr_cache_bytes -= h->csr_cache.back().host_bytes();
    h->csr_cache.pop_back();
  }
  return h->csr_cache.front().plan;
}

}  // namespace cfm
