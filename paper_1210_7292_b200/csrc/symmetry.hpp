// Host+device restatement of the reference's symmetry machinery.
//
//   canonicalize            symmetry.py:63-75   (flips = t_i < 0; stable sort of
//                                                axes by (-|t_i|, i), 1-based)
//   permutation_index_table symmetry.py:86-102  (flip comps, then reorder,
//                                                then flatten a1 + a2 l + a3 l^2)
//   inverse_permutation_table symmetry.py:105-111
//   far condition           octree.py:64-65     (t.t > 3)
//
// Transfer vectors are addressed by a t-code in [0, 343); permutation specs by
// a perm id in [0, 48) = flipmask * 6 + rank of axis_order.
#pragma once
#include <cstdint>
#include <vector>

namespace cfm {

constexpr int kNumCodes = 343;
constexpr int kNumPerms = 48;

#if defined(__CUDACC__)
#define CFM_HD __host__ __device__ inline
#else
#define CFM_HD inline
#endif

CFM_HD int tcode(int t0, int t1, int t2) { return (t0 + 3) * 49 + (t1 + 3) * 7 + (t2 + 3); }
CFM_HD void tcode_decode(int c, int& t0, int& t1, int& t2) {
  t0 = c / 49 - 3;
  t1 = (c / 7) % 7 - 3;
  t2 = c % 7 - 3;
}
CFM_HD bool is_far(int t0, int t1, int t2) { return t0 * t0 + t1 * t1 + t2 * t2 > 3; }

// Axis orders in lexicographic order; index = perm id % 6.
CFM_HD void axis_order_of(int k, int o[3]) {
  const int tab[6][3] = {{1, 2, 3}, {1, 3, 2}, {2, 1, 3}, {2, 3, 1}, {3, 1, 2}, {3, 2, 1}};
  o[0] = tab[k][0]; o[1] = tab[k][1]; o[2] = tab[k][2];
}
CFM_HD int axis_order_rank(const int o[3]) {
  // rank among the 6 permutations of (1,2,3) in lexicographic order
  return (o[0] - 1) * 2 + ((o[1] > o[2]) ? 1 : 0);
}

// canonicalize(t) -> (t_sym, perm id).  Stable descending sort of |t| with the
// tie-break on the original axis index, exactly as sorted(range(3),
// key=lambda i: (-abs_t[i], i)).
CFM_HD void canonicalize(int t0, int t1, int t2, int tsym[3], int& perm_id) {
  const int t[3] = {t0, t1, t2};
  int a[3] = {t0 < 0 ? -t0 : t0, t1 < 0 ? -t1 : t1, t2 < 0 ? -t2 : t2};
  int idx[3] = {0, 1, 2};
  // insertion sort (stable) on key (-a[i], i)
  for (int i = 1; i < 3; ++i) {
    int v = idx[i];
    int j = i - 1;
    while (j >= 0 && (a[idx[j]] < a[v] || (a[idx[j]] == a[v] && idx[j] > v))) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = v;
  }
  int o[3] = {idx[0] + 1, idx[1] + 1, idx[2] + 1};
  for (int i = 0; i < 3; ++i) tsym[i] = a[idx[i]];
  int flips = (t[0] < 0 ? 1 : 0) | (t[1] < 0 ? 2 : 0) | (t[2] < 0 ? 4 : 0);
  perm_id = flips * 6 + axis_order_rank(o);
}

// table[j] for a perm id and order l (0-based flat positions).
inline std::vector<int> permutation_table(int perm_id, int order) {
  const int n = order * order * order;
  std::vector<int> table(n);
  const int flips = perm_id / 6;
  int o[3];
  axis_order_of(perm_id % 6, o);
  for (int j = 0; j < n; ++j) {
    int c[3] = {j % order, (j / order) % order, j / (order * order)};
    for (int ax = 0; ax < 3; ++ax)
      if (flips & (1 << ax)) c[ax] = order - 1 - c[ax];
    const int r0 = c[o[0] - 1], r1 = c[o[1] - 1], r2 = c[o[2] - 1];
    table[j] = r0 + r1 * order + r2 * order * order;
  }
  return table;
}

inline std::vector<int> inverse_table(const std::vector<int>& table) {
  std::vector<int> inv(table.size());
  for (size_t j = 0; j < table.size(); ++j) inv[table[j]] = int(j);
  return inv;
}

// The 16 cone representatives of the full 316-vector far field, sorted
// lexicographically (SymmetryMap.cone of the full list, symmetry.py:133).
inline std::vector<int> full_cone_codes() {
  std::vector<int> out;
  for (int a = 0; a <= 3; ++a)
    for (int b = 0; b <= a; ++b)
      for (int c = 0; c <= b; ++c)
        if (is_far(a, b, c)) out.push_back(tcode(a, b, c));
  return out;  // tcode order == lexicographic order of (a, b, c)
}

}  // namespace cfm
