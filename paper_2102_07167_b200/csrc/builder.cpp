// builder.cpp — host-side block builder behind kur_graph_build (product code).
//
// Steps:
//  1. validate the row-segmented pattern (error conventions of include/kur.h);
//  2. per block (row community a x column community b) count the ones over
//     the off-diagonal entries and decide DENSE iff zeros < ones (P:96, P:14,
//     P:538-544; tie -> SPARSE, reading R3) or the caller's threshold;
//     D(a) = dense column communities of a (block sums precomputed);
//  3. internal numbering = communities contiguous, rows of a
//     community by decreasing list length;
//  4. cut community-aligned tiles, pick hot windows per tile, emit the
//     complement lists Z_j (dense blocks, subtracted) and the
//     non-zero lists NZ_j (sparse blocks, added) in the chunked
//     16-bit / 32-bit layout of plan.h.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <array>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>
#include <numeric>
#include <omp.h>

#include "plan.h"

namespace kur {
namespace {

struct Err {
  std::mutex mu;
  int64_t where = INT64_MAX;
  kur_status st = KUR_OK;
  std::string msg;
  void set(int64_t w, kur_status s, const std::string& m) {
    std::lock_guard<std::mutex> g(mu);
    if (w < where) { where = w; st = s; msg = m; }
  }
};

struct Src {  // the caller's description plus derived community data
  const kur_graph_desc* d;
  int64_t n;
  int32_t C;
  std::vector<int64_t> moff;   // members offsets [C+1]
  std::vector<int32_t> mem;    // members (ascending user id)
  std::vector<int64_t> csize;  // community sizes
  std::vector<uint8_t> dense;  // only via D lists; per-community bitmap built on demand
};

inline bool has_diag(const int32_t* lst, int64_t len, int32_t u) {
  return std::binary_search(lst, lst + len, u);
}

// Enumerate the stored entries of user row u (community a) after the
// dense/sparse decision: cb(user_col, neg) with neg = 1 for complement
// (subtracted) entries and 0 for non-zero entries.  Segment order, ascending
// within a segment.
template <class F>
void enumerate_row(const Src& S, const std::vector<int32_t>& D_ptr, const std::vector<int32_t>& D_idx,
                   int32_t u, F cb) {
  const kur_graph_desc* d = S.d;
  const int32_t a = d->community[u];
  int64_t s = d->seg_ptr[u];
  const int64_t s1 = d->seg_ptr[u + 1];
  int32_t di = D_ptr[a];
  const int32_t d1 = D_ptr[a + 1];
  while (s < s1 || di < d1) {
    const int32_t bs = s < s1 ? d->seg_comm[s] : INT32_MAX;
    const int32_t bd = di < d1 ? D_idx[di] : INT32_MAX;
    const int32_t b = std::min(bs, bd);
    const bool dense = (bd == b);
    const bool seg = (bs == b);
    const int32_t* lst = seg ? d->idx + d->idx_ptr[s] : nullptr;
    const int64_t len = seg ? d->idx_ptr[s + 1] - d->idx_ptr[s] : 0;
    const int kind = seg ? d->seg_kind[s] : -1;
    const int32_t* m = S.mem.data() + S.moff[b];
    const int64_t nm = S.moff[b + 1] - S.moff[b];
    auto complement = [&](int neg) {  // members of b minus lst minus u
      int64_t z = 0;
      for (int64_t e = 0; e < nm; ++e) {
        const int32_t k = m[e];
        while (z < len && lst[z] < k) ++z;
        if (z < len && lst[z] == k) continue;
        if (k != u) cb(k, neg);
      }
    };
    if (dense) {
      if (seg && kind == KUR_ZEROS) {
        for (int64_t e = 0; e < len; ++e) if (lst[e] != u) cb(lst[e], 1);
      } else {
        complement(1);  // ONES segment or no segment: zeros = complement
      }
    } else if (seg) {
      if (kind == KUR_ONES) {
        for (int64_t e = 0; e < len; ++e) if (lst[e] != u) cb(lst[e], 0);
      } else {
        complement(0);
      }
    }
    if (seg) ++s;
    if (dense) ++di;
  }
}


// Form the chunks of a hot part.  Rows (ord, longest first) are taken in
// pools of 256; each pool is split greedily into 32 quarter-warps of 8 rows
// whose per-residue totals (slot mod 8) are balanced, because a quarter's
// conflict-free schedule needs max(longest row, largest residue total)
// positions; a local search then swaps rows between quarters while the sum of
// the two bounds drops; quarters are sorted by their bound and grouped 4 per
// chunk.  (Config-5-like SBM: hot padding 13.7 % -> 6.2 %, with the 4-slot
// half-group tail of plan.h.)
//
// Rows split into w = 2^lp pieces (row pieces, w <= 8) are packed as items of w adjacent, aligned
// lanes: a quarter then holds 8 / w rows, an item's lane length is its longest piece (cnt), its
// residue counts are the whole row's; `ord` entries are item ids and the returned lanes hold
// item ids at the first lane of each item (the caller expands them to pieces).
template <class CountFn>
void plan_pools(const std::vector<int32_t>& ord, const std::vector<int32_t>& cnt,
                std::vector<std::array<int32_t, 32>>& lanes, CountFn count, int w = 1) {
  constexpr int POOL = 256, NQ = POOL / 8;
  const int per_q = 8 / w;            // items per quarter
  const int pool_items = NQ * per_q;  // items per pool (256 lanes)
  for (size_t p0 = 0; p0 < ord.size(); p0 += (size_t)pool_items) {
    const int np = (int)std::min<size_t>((size_t)pool_items, ord.size() - p0);
    const int nq = (np + per_q - 1) / per_q;
    int cv[POOL][8];
    std::memset(cv, 0, sizeof(cv));
    for (int i = 0; i < np; ++i) count(ord[p0 + (size_t)i], cv[i]);
    int qt[NQ][8], qf[NQ], qlen[NQ], qm[NQ][8], qi[NQ][8];
    std::memset(qt, 0, sizeof(qt));
    std::memset(qf, 0, sizeof(qf));
    std::memset(qlen, 0, sizeof(qlen));
    for (int i = 0; i < np; ++i) {
      int bq = -1;
      long bmx = 0, bss = 0;
      for (int q = 0; q < nq; ++q) {
        if (qf[q] == per_q) continue;
        long mx = std::max(qlen[q], cnt[(size_t)ord[p0 + (size_t)i]]), ss = 0;
        for (int r = 0; r < 8; ++r) {
          const long v = qt[q][r] + cv[i][r];
          mx = std::max(mx, v);
          ss += v * v;
        }
        if (bq < 0 || mx < bmx || (mx == bmx && ss < bss)) { bq = q; bmx = mx; bss = ss; }
      }
      for (int r = 0; r < 8; ++r) qt[bq][r] += cv[i][r];
      qlen[bq] = std::max(qlen[bq], cnt[(size_t)ord[p0 + (size_t)i]]);
      qi[bq][qf[bq]] = i;
      qm[bq][qf[bq]++] = ord[p0 + (size_t)i];
    }
    // local search: swap two rows of different quarters while it lowers the sum of
    // the two quarters' bounds (only residue-limited quarters can gain)
    auto rlen = [&](int i) { return cnt[(size_t)ord[p0 + (size_t)i]]; };
    auto qbound = [&](int q) {
      int b = qlen[q];
      for (int r = 0; r < 8; ++r) b = std::max(b, qt[q][r]);
      return b;
    };
    for (int pass = 0; pass < 3; ++pass) {
      bool any = false;
      for (int q = 0; q < nq; ++q) {
        const int bq = qbound(q);
        if (bq == qlen[q]) continue;
        int rs = 0;
        for (int r = 1; r < 8; ++r)
          if (qt[q][r] > qt[q][rs]) rs = r;
        int best = 0, bm = -1, bq2 = -1, bm2 = -1;
        for (int m = 0; m < qf[q]; ++m) {
          const int i = qi[q][m];
          for (int q2 = 0; q2 < nq; ++q2) {
            if (q2 == q) continue;
            const int b2 = qbound(q2);
            for (int m2 = 0; m2 < qf[q2]; ++m2) {
              const int j = qi[q2][m2];
              if (qt[q][rs] - cv[i][rs] + cv[j][rs] >= bq) continue;  // the worst residue must drop
              int l1 = rlen(j), l2 = rlen(i);
              for (int k = 0; k < qf[q]; ++k) if (k != m) l1 = std::max(l1, rlen(qi[q][k]));
              for (int k = 0; k < qf[q2]; ++k) if (k != m2) l2 = std::max(l2, rlen(qi[q2][k]));
              int n1 = l1, n2 = l2;
              for (int r = 0; r < 8; ++r) {
                n1 = std::max(n1, qt[q][r] - cv[i][r] + cv[j][r]);
                n2 = std::max(n2, qt[q2][r] - cv[j][r] + cv[i][r]);
              }
              const int gain = bq + b2 - n1 - n2;
              if (gain > best) { best = gain; bm = m; bq2 = q2; bm2 = m2; }
            }
          }
        }
        if (bm < 0) continue;
        const int i = qi[q][bm], j = qi[bq2][bm2];
        for (int r = 0; r < 8; ++r) {
          qt[q][r] += cv[j][r] - cv[i][r];
          qt[bq2][r] += cv[i][r] - cv[j][r];
        }
        qi[q][bm] = j;
        qm[q][bm] = ord[p0 + (size_t)j];
        qi[bq2][bm2] = i;
        qm[bq2][bm2] = ord[p0 + (size_t)i];
        qlen[q] = 0;
        qlen[bq2] = 0;
        for (int k = 0; k < qf[q]; ++k) qlen[q] = std::max(qlen[q], rlen(qi[q][k]));
        for (int k = 0; k < qf[bq2]; ++k) qlen[bq2] = std::max(qlen[bq2], rlen(qi[bq2][k]));
        any = true;
      }
      if (!any) break;
    }
    int qord[NQ], qb[NQ];
    for (int q = 0; q < nq; ++q) {
      qord[q] = q;
      qb[q] = qlen[q];
      for (int r = 0; r < 8; ++r) qb[q] = std::max(qb[q], qt[q][r]);
    }
    std::sort(qord, qord + nq, [&](int x, int y) { return qb[x] > qb[y]; });
    for (int c = 0; c * 4 < nq; ++c) {
      std::array<int32_t, 32> a;
      a.fill(-1);
      for (int k = 0; k < 4 && c * 4 + k < nq; ++k) {
        const int q = qord[c * 4 + k];
        for (int m = 0; m < qf[q]; ++m) a[(size_t)(k * 8 + m * w)] = qm[q][m];
      }
      lanes.push_back(a);
    }
  }
}

// Schedule the entries of one quarter-warp (lst[lane][residue] = window slots)
// into positions of 8 slots with pairwise distinct residues (one 16-byte bank
// group per lane: conflict-free LDS.128).  Bipartite edge colouring of the
// lane x residue multigraph: at each position a matching that covers every
// "critical" lane / residue (remaining degree = remaining positions), found
// with augmenting paths, so the schedule length stays at the lower bound
// max(lane length, residue total) (Koenig's edge-colouring theorem).
// Unused lanes of a position get the zero sentinel of a free residue.
void schedule_quarter(std::vector<uint16_t> (&lst)[8][8], std::vector<uint32_t>& P8) {
  P8.clear();
  int c8[8][8], rem[8] = {0}, tot[8] = {0};
  for (int l = 0; l < 8; ++l)
    for (int r = 0; r < 8; ++r) {
      c8[l][r] = (int)lst[l][r].size();
      rem[l] += c8[l][r];
      tot[r] += c8[l][r];
    }
  int Lb = 0;
  for (int i = 0; i < 8; ++i) Lb = std::max(Lb, std::max(rem[i], tot[i]));
  int asg[8], owner[8], adj[8];
  std::function<bool(int, int&, int)> aug_lane = [&](int x, int& seen, int crit_r) -> bool {
    // residues: critical first, then by remaining total (scarce residues are the bottleneck)
    int order[8];
    for (int r = 0; r < 8; ++r) order[r] = r;
    std::sort(order, order + 8, [&](int u, int v) {
      const int cu = (crit_r >> u) & 1, cvv = (crit_r >> v) & 1;
      if (cu != cvv) return cu > cvv;
      return tot[u] > tot[v];
    });
    for (int k = 0; k < 8; ++k) {
      const int r = order[k];
      if (!((adj[x] >> r) & 1) || ((seen >> r) & 1)) continue;
      seen |= 1 << r;
      if (owner[r] < 0 || aug_lane(owner[r], seen, crit_r)) { owner[r] = x; asg[x] = r; return true; }
    }
    return false;
  };
  std::function<bool(int, int&)> aug_res = [&](int y, int& seenl) -> bool {
    for (int x = 0; x < 8; ++x) {
      if (!((adj[x] >> y) & 1) || ((seenl >> x) & 1)) continue;
      seenl |= 1 << x;
      if (asg[x] < 0 || aug_res(asg[x], seenl)) { asg[x] = y; owner[y] = x; return true; }
    }
    return false;
  };
  for (int pos = 0;; ++pos) {
    int any = 0;
    for (int l = 0; l < 8; ++l) any |= rem[l];
    if (!any) break;
    const int R = std::max(Lb - pos, 1);
    int crit_l = 0, crit_r = 0;
    for (int i = 0; i < 8; ++i) {
      if (rem[i] >= R) crit_l |= 1 << i;
      if (tot[i] >= R) crit_r |= 1 << i;
      asg[i] = owner[i] = -1;
      adj[i] = 0;
      for (int r = 0; r < 8; ++r)
        if (c8[i][r] > 0) adj[i] |= 1 << r;
    }
    int lord[8];
    for (int i = 0; i < 8; ++i) lord[i] = i;
    std::sort(lord, lord + 8, [&](int u, int v) { return rem[u] > rem[v]; });
    for (int k = 0; k < 8; ++k) {  // 1) critical lanes
      const int x = lord[k];
      if ((crit_l >> x) & 1) { int seen = 0; aug_lane(x, seen, crit_r); }
    }
    for (int y = 0; y < 8; ++y)  // 2) critical residues (never unmatches a lane)
      if (((crit_r >> y) & 1) && owner[y] < 0) { int seenl = 0; aug_res(y, seenl); }
    for (int k = 0; k < 8; ++k) {  // 3) everybody else, longest first
      const int x = lord[k];
      if (rem[x] && asg[x] < 0) { int seen = 0; aug_lane(x, seen, crit_r); }
    }
    int used = 0;
    for (int l = 0; l < 8; ++l)
      if (asg[l] >= 0) used |= 1 << asg[l];
    for (int l = 0; l < 8; ++l) {
      uint32_t v;
      if (asg[l] >= 0) {
        const int r = asg[l];
        v = lst[l][r].back();
        lst[l][r].pop_back();
        c8[l][r]--;
        rem[l]--;
        tot[r]--;
      } else {
        int r = 0;
        while ((used >> r) & 1) ++r;
        used |= 1 << r;
        v = HOT_SENT + (uint32_t)r;
      }
      P8.push_back(v);
    }
  }
}

}  // namespace

kur_status build_plan(const kur_graph_desc* d, int32_t rank, int32_t world, int sm_count,
                      HostPlan& P, std::string& err) {
  // ------------------------------------------------------------ 1. validate
  if (!d || d->n < 1 || d->n_comm < 1 || !d->community || !d->seg_ptr || !d->idx_ptr) {
    err = "kur_graph_desc: n >= 1, n_comm >= 1 and non-NULL community/seg_ptr/idx_ptr required";
    return KUR_ERR_INVALID_ARG;
  }
  if (d->n >= INT32_MAX - 2 * WZ) { err = "n too large for int32 internal ids"; return KUR_ERR_UNSUPPORTED; }
  if (d->scaling != KUR_SCALING_UNIFORM && d->scaling != KUR_SCALING_DEGREE) {
    err = "scaling must be KUR_SCALING_UNIFORM or KUR_SCALING_DEGREE";
    return KUR_ERR_INVALID_ARG;
  }
  if (d->reserved != 0) { err = "reserved must be 0"; return KUR_ERR_INVALID_ARG; }
  const int force_rows = d->flags & 0xFFFF;
  const int force_split = (d->flags >> 16) & 3;  // KUR_FLAG_REMOTE_PASS (1) / KUR_FLAG_REMOTE_INLINE (2)
  if ((force_rows != 0 && (force_rows < 32 || force_rows > MAX_TILE_ROWS || force_rows % 32 != 0)) ||
      (d->flags >> 18) != 0 || force_split == 3) {
    err = "flags: 0 or a tile size in rows (multiple of 32 in [32, 2048]), optionally | KUR_FLAG_REMOTE_PASS "
          "or | KUR_FLAG_REMOTE_INLINE";
    return KUR_ERR_INVALID_ARG;
  }
  const double thr = d->dense_threshold;
  if (std::isnan(thr) || thr > 1.0) { err = "dense_threshold must be <= 1 (or < 0 for the paper rule)"; return KUR_ERR_INVALID_ARG; }
  if (world < 1 || rank < 0 || rank >= world) { err = "bad rank/world"; return KUR_ERR_INVALID_ARG; }
  const int64_t n = d->n;
  const int32_t C = d->n_comm;
  if (d->seg_ptr[0] != 0) { err = "seg_ptr[0] must be 0"; return KUR_ERR_SIZE_MISMATCH; }
  const int64_t nseg = d->seg_ptr[n];
  if (nseg < 0) { err = "seg_ptr[n] < 0"; return KUR_ERR_SIZE_MISMATCH; }
  if (nseg > 0 && (!d->seg_comm || !d->seg_kind)) { err = "seg_comm/seg_kind NULL"; return KUR_ERR_INVALID_ARG; }
  if (d->idx_ptr[0] != 0) { err = "idx_ptr[0] must be 0"; return KUR_ERR_SIZE_MISMATCH; }
  if (d->idx_ptr[nseg] > 0 && !d->idx) { err = "idx NULL"; return KUR_ERR_INVALID_ARG; }
  Err E;
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < n; ++u) {
    if (d->community[u] < 0 || d->community[u] >= C)
      E.set(u, KUR_ERR_PARTITION, "community label of node " + std::to_string(u) + " outside [0, n_comm)");
  }
  if (E.st != KUR_OK) { err = E.msg; return E.st; }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t u = 0; u < n; ++u) {
    const int64_t s0 = d->seg_ptr[u], s1 = d->seg_ptr[u + 1];
    if (s1 < s0 || s1 > nseg) { E.set(u, KUR_ERR_SIZE_MISMATCH, "seg_ptr not monotone at row " + std::to_string(u)); continue; }
    int32_t pb = -1;
    for (int64_t s = s0; s < s1; ++s) {
      const int32_t b = d->seg_comm[s];
      if (b < 0 || b >= C) { E.set(u, KUR_ERR_PARTITION, "seg_comm outside [0, n_comm) in row " + std::to_string(u)); break; }
      if (b == pb) { E.set(u, KUR_ERR_DUPLICATE_INDEX, "community given two segments in row " + std::to_string(u)); break; }
      if (b < pb) { E.set(u, KUR_ERR_INVALID_ARG, "seg_comm not increasing in row " + std::to_string(u)); break; }
      pb = b;
      if (d->seg_kind[s] > 1) { E.set(u, KUR_ERR_INVALID_ARG, "bad seg_kind in row " + std::to_string(u)); break; }
      const int64_t i0 = d->idx_ptr[s], i1 = d->idx_ptr[s + 1];
      if (i1 < i0) { E.set(u, KUR_ERR_SIZE_MISMATCH, "idx_ptr not monotone in row " + std::to_string(u)); break; }
      int64_t pk = -1;
      bool bad = false;
      for (int64_t e = i0; e < i1; ++e) {
        const int32_t k = d->idx[e];
        if (k < 0 || k >= n) { E.set(u, KUR_ERR_INDEX_RANGE, "column id outside [0, n) in row " + std::to_string(u)); bad = true; break; }
        if (d->community[k] != b) { E.set(u, KUR_ERR_PARTITION, "column outside its segment's community in row " + std::to_string(u)); bad = true; break; }
        if (k == pk) { E.set(u, KUR_ERR_DUPLICATE_INDEX, "column listed twice in row " + std::to_string(u)); bad = true; break; }
        if (k < pk) { E.set(u, KUR_ERR_INVALID_ARG, "segment list not ascending in row " + std::to_string(u)); bad = true; break; }
        pk = k;
      }
      if (bad) break;
    }
  }
  if (E.st != KUR_OK) { err = E.msg; return E.st; }

  // ------------------------------------------------------------ communities
  Src S;
  S.d = d;
  S.n = n;
  S.C = C;
  S.moff.assign((size_t)C + 1, 0);
  for (int64_t u = 0; u < n; ++u) S.moff[(size_t)d->community[u] + 1]++;
  for (int32_t c = 0; c < C; ++c) S.moff[(size_t)c + 1] += S.moff[(size_t)c];
  S.csize.resize((size_t)C);
  for (int32_t c = 0; c < C; ++c) S.csize[(size_t)c] = S.moff[(size_t)c + 1] - S.moff[(size_t)c];
  S.mem.resize((size_t)n);
  {
    std::vector<int64_t> fill(S.moff.begin(), S.moff.end() - 1);
    for (int64_t u = 0; u < n; ++u) S.mem[(size_t)fill[(size_t)d->community[u]]++] = (int32_t)u;
  }

  // ------------------------------------------------------------ 2. census + rule
  std::vector<std::vector<int32_t>> Dl((size_t)C);
  std::atomic<int64_t> nnz{0}, ndense{0}, nsparse{0};
#pragma omp parallel
  {
    std::vector<int64_t> ones((size_t)C, 0);
    std::vector<uint8_t> seen((size_t)C, 0);
    std::vector<int32_t> touched;
#pragma omp for schedule(dynamic, 1)
    for (int32_t a = 0; a < C; ++a) {
      touched.clear();
      for (int64_t mi = S.moff[(size_t)a]; mi < S.moff[(size_t)a + 1]; ++mi) {
        const int32_t u = S.mem[(size_t)mi];
        for (int64_t s = d->seg_ptr[u]; s < d->seg_ptr[u + 1]; ++s) {
          const int32_t b = d->seg_comm[s];
          const int32_t* lst = d->idx + d->idx_ptr[s];
          const int64_t len = d->idx_ptr[s + 1] - d->idx_ptr[s];
          const int64_t lnd = len - ((b == a && has_diag(lst, len, u)) ? 1 : 0);
          const int64_t o = d->seg_kind[s] == KUR_ONES ? lnd : S.csize[(size_t)b] - (b == a ? 1 : 0) - lnd;
          if (!seen[(size_t)b]) { seen[(size_t)b] = 1; touched.push_back(b); }
          ones[(size_t)b] += o;
        }
      }
      std::sort(touched.begin(), touched.end());
      int64_t lnnz = 0, ld = 0, ls = 0;
      for (int32_t b : touched) {
        const int64_t na = S.csize[(size_t)a], nb = S.csize[(size_t)b];
        const int64_t total = na * nb - (a == b ? na : 0);
        const int64_t o = ones[(size_t)b];
        const int64_t z = total - o;
        bool dense;
        if (thr < 0) dense = z < o;  // paper rule P:96 (tie -> sparse)
        else dense = (double)z < thr * (double)total;
        if (total == 0) dense = false;
        if (dense) { Dl[(size_t)a].push_back(b); ++ld; }
        else if (o > 0) ++ls;
        lnnz += o;
        ones[(size_t)b] = 0;
        seen[(size_t)b] = 0;
      }
      nnz += lnnz;
      ndense += ld;
      nsparse += ls;
    }
  }
  P.D_ptr.assign((size_t)C + 1, 0);
  for (int32_t a = 0; a < C; ++a) P.D_ptr[(size_t)a + 1] = P.D_ptr[(size_t)a] + (int32_t)Dl[(size_t)a].size();
  P.D_idx.clear();
  for (int32_t a = 0; a < C; ++a) P.D_idx.insert(P.D_idx.end(), Dl[(size_t)a].begin(), Dl[(size_t)a].end());

  // ------------------------------------------------------------ 3. lengths + order
  std::vector<int64_t> rlen((size_t)n, 0), ones_off((size_t)n, 0);
  std::vector<uint8_t> selfl((size_t)n, 0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t u = 0; u < n; ++u) {
    const int32_t a = d->community[u];
    int64_t s = d->seg_ptr[u];
    const int64_t s1 = d->seg_ptr[u + 1];
    int32_t di = P.D_ptr[(size_t)a];
    const int32_t d1 = P.D_ptr[(size_t)a + 1];
    int64_t L = 0, ones = 0;
    for (int64_t t = s; t < s1; ++t) {  // degree: off-diagonal ones, and a listed self-loop (R22)
      const int32_t b = d->seg_comm[t];
      const int32_t* lst = d->idx + d->idx_ptr[t];
      const int64_t len = d->idx_ptr[t + 1] - d->idx_ptr[t];
      const bool diag = b == a && has_diag(lst, len, (int32_t)u);
      const int64_t lnd = len - (diag ? 1 : 0);
      if (d->seg_kind[t] == KUR_ONES) {
        ones += lnd;
        if (diag) selfl[(size_t)u] = 1;
      } else {
        ones += S.csize[(size_t)b] - (b == a ? 1 : 0) - lnd;
      }
    }
    ones_off[(size_t)u] = ones;
    while (s < s1 || di < d1) {
      const int32_t bs = s < s1 ? d->seg_comm[s] : INT32_MAX;
      const int32_t bd = di < d1 ? P.D_idx[(size_t)di] : INT32_MAX;
      const int32_t b = std::min(bs, bd);
      const bool dense = bd == b, seg = bs == b;
      const int64_t nb_off = S.csize[(size_t)b] - (b == a ? 1 : 0);
      int64_t lnd = 0;
      int kind = -1;
      if (seg) {
        const int32_t* lst = d->idx + d->idx_ptr[s];
        const int64_t len = d->idx_ptr[s + 1] - d->idx_ptr[s];
        lnd = len - ((b == a && has_diag(lst, len, (int32_t)u)) ? 1 : 0);
        kind = d->seg_kind[s];
      }
      if (dense) L += (seg && kind == KUR_ZEROS) ? lnd : nb_off - lnd;
      else if (seg) L += kind == KUR_ONES ? lnd : nb_off - lnd;
      if (seg) ++s;
      if (dense) ++di;
    }
    rlen[(size_t)u] = L;
  }
  P.n = n;
  P.C = C;
  P.rank = rank;
  P.world = world;
  P.nnz = nnz.load();
  P.n_dense_blocks = ndense.load();
  P.n_sparse_blocks = nsparse.load();
  P.perm.resize((size_t)n);
  P.comm_off.assign((size_t)C + 1, 0);
  for (int32_t c = 0; c <= C; ++c) P.comm_off[(size_t)c] = (int32_t)S.moff[(size_t)c];
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t a = 0; a < C; ++a) {
    int32_t* p = P.perm.data() + S.moff[(size_t)a];
    const int64_t na = S.csize[(size_t)a];
    std::copy(S.mem.begin() + S.moff[(size_t)a], S.mem.begin() + S.moff[(size_t)a + 1], p);
    std::stable_sort(p, p + na, [&](int32_t x, int32_t y) { return rlen[(size_t)x] > rlen[(size_t)y]; });
  }
  std::vector<int32_t> inv((size_t)n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) inv[(size_t)P.perm[(size_t)i]] = (int32_t)i;

  // ------------------------------------------------------------ 4. tiles
  // The largest power-of-two tile (256..2048 rows) that still gives >= 4
  // tiles per SM (measured on B200: smaller tiles leave warps idle per part,
  // larger ones unbalance heterogeneous graphs).  Tiny graphs run whole
  // trajectories in one CTA (kur_step) with one tile.
  int64_t total_len = 0;
#pragma omp parallel for reduction(+ : total_len)
  for (int64_t u = 0; u < n; ++u) total_len += rlen[(size_t)u];
  // Every tile rule below depends on the graph (and the SM count) only, never on the world
  // size or rank: tiles, their parts and the fixed reduction order are then the same at every
  // world size, which makes results bitwise independent of the sharding.
  const bool tiny = n <= 8192 && total_len <= (1 << 18);
  P.small = world == 1 && tiny;
  // no stored entries (complete graphs: one dense block, empty complement lists) -> no shared
  // memory and nothing to balance: the largest tiles amortise the per-CTA latency (config 2:
  // 25.7 -> 21.5 us per stage with 2048- instead of 1024-row tiles, see the commit for 4096)
  // Their tile is sized so the tiles fill exactly one wave of 2 CTAs per SM (config 2: 296
  // tiles of 3552 rows instead of 256 of 4096, which left 40 SMs with one CTA).
  int rows_per_tile = force_rows ? force_rows : tiny ? MAX_TILE_ROWS : 0;
  if (!rows_per_tile && total_len == 0) {
    const int64_t per = (n + 2LL * sm_count - 1) / (2LL * sm_count);
    rows_per_tile = (int)std::min<int64_t>(MAX_TILE_ROWS_NOPARTS, std::max<int64_t>(256, (per + 31) / 32 * 32));
  }
  for (int r = MAX_TILE_ROWS; r >= 256 && !rows_per_tile; r >>= 1) {
    int64_t nt = 0;
    for (int32_t c = 0; c < C; ++c) nt += (S.csize[(size_t)c] + r - 1) / r;
    if (nt >= 4LL * sm_count || r == 256) rows_per_tile = r;
  }
  // One partial wave: when even 256-row tiles give fewer tiles than one wave of 2 CTAs per SM
  // (config 3: 256 tiles for 296 slots, so 108 SMs ran two tiles and 40 ran one), each community
  // is cut into floor(2 SMs x size / N) tiles of equal size instead (config 3: 18 tiles of 227-228
  // rows, 288 tiles, every SM at most 2 x 228 rows instead of 2 x 256); never fewer tiles than
  // the 256-row rule, never more than one wave, never below 192 rows per tile.
  std::vector<int32_t> ctiles((size_t)C, 0);  // > 0: balanced split into that many tiles
  if (!force_rows && !tiny && total_len > 0 && rows_per_tile == 256) {
    const int64_t T = 2LL * sm_count;
    int64_t nt256 = 0, ntb = 0;
    for (int32_t c = 0; c < C; ++c) nt256 += (S.csize[(size_t)c] + 255) / 256;
    if (nt256 < T) {
      for (int32_t c = 0; c < C; ++c) {
        const int64_t sz = S.csize[(size_t)c];
        if (sz == 0) continue;
        // (tiles of >= 192 rows: a graph far smaller than one wave keeps ~256-row tiles, only balanced)
        ctiles[(size_t)c] = (int32_t)std::max<int64_t>((sz + 255) / 256, std::min<int64_t>(T * sz / n, sz / 192));
        ntb += ctiles[(size_t)c];
      }
      if (ntb > T) std::fill(ctiles.begin(), ctiles.end(), 0);
    }
  }
  P.rows_per_tile = rows_per_tile;
  std::vector<int32_t> crt((size_t)C, rows_per_tile);
  std::vector<TileDesc> all;
  P.comm_tile0.assign((size_t)C + 1, 0);
  for (int32_t c = 0; c < C; ++c) {
    P.comm_tile0[(size_t)c] = (int32_t)all.size();
    const int RT = crt[(size_t)c];
    if (ctiles[(size_t)c] > 0) {  // balanced split
      const int64_t sz = S.csize[(size_t)c], k = ctiles[(size_t)c];
      for (int64_t i = 0; i < k; ++i) {
        TileDesc t{};
        t.row0 = (int32_t)(S.moff[(size_t)c] + sz * i / k);
        t.nrows = (int32_t)(S.moff[(size_t)c] + sz * (i + 1) / k - t.row0);
        t.comm = c;
        all.push_back(t);
      }
      continue;
    }
    for (int64_t r0 = S.moff[(size_t)c]; r0 < S.moff[(size_t)c + 1]; r0 += RT) {
      TileDesc t{};
      t.row0 = (int32_t)r0;
      t.nrows = (int32_t)std::min<int64_t>(RT, S.moff[(size_t)c + 1] - r0);
      t.comm = c;
      all.push_back(t);
    }
  }
  P.comm_tile0[(size_t)C] = (int32_t)all.size();
  const int64_t ntiles_all = (int64_t)all.size();
  // per-tile work estimate (entries), then shards of whole communities
  std::vector<int64_t> twork((size_t)ntiles_all, 0);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < ntiles_all; ++t) {
    int64_t w = 0;
    for (int32_t r = 0; r < all[(size_t)t].nrows; ++r) w += rlen[(size_t)P.perm[(size_t)(all[(size_t)t].row0 + r)]] + 8;
    twork[(size_t)t] = w;
  }
  std::vector<int64_t> cwork((size_t)C, 0);
  for (int32_t c = 0; c < C; ++c)
    for (int32_t t = P.comm_tile0[(size_t)c]; t < P.comm_tile0[(size_t)c + 1]; ++t) cwork[(size_t)c] += twork[(size_t)t];
  // Shards: contiguous tile ranges balanced by work.  Whole communities per rank when that
  // balances (then a tile's own-community windows are always local: phase A overlaps the
  // exchange); otherwise (few large communities, e.g. one complete graph) the
  // boundaries fall between tiles inside communities.  Every rank computes the same boundaries.
  std::vector<int32_t> tile_b((size_t)world + 1, 0);
  {
    const double totw = (double)std::accumulate(twork.begin(), twork.end(), (int64_t)0);
    auto max_shard = [&](const std::vector<int32_t>& b) {
      int64_t m = 0;
      for (int32_t r = 0; r < world; ++r) {
        int64_t w = 0;
        for (int32_t t = b[(size_t)r]; t < b[(size_t)r + 1]; ++t) w += twork[(size_t)t];
        m = std::max(m, w);
      }
      return m;
    };
    std::vector<int32_t> cb((size_t)world + 1, 0), tb((size_t)world + 1, 0);
    int64_t acc = 0;
    int32_t c = 0;
    for (int32_t r = 1; r < world; ++r) {  // community granularity
      const double target = totw * r / world;
      while (c < C && (double)(acc + cwork[(size_t)c] / 2) < target) acc += cwork[(size_t)c++];
      cb[(size_t)r] = P.comm_tile0[(size_t)std::max<int32_t>(c, 0)];
      cb[(size_t)r] = std::max(cb[(size_t)r], cb[(size_t)r - 1]);
    }
    cb[(size_t)world] = (int32_t)ntiles_all;
    acc = 0;
    int32_t t = 0;
    for (int32_t r = 1; r < world; ++r) {  // tile granularity
      const double target = totw * r / world;
      while (t < ntiles_all && (double)(acc + twork[(size_t)t] / 2) < target) acc += twork[(size_t)t++];
      tb[(size_t)r] = std::max(t, tb[(size_t)r - 1]);
    }
    tb[(size_t)world] = (int32_t)ntiles_all;
    tile_b = (double)max_shard(cb) <= 1.1 * (double)max_shard(tb) ? cb : tb;
  }
  P.shard_row0.resize((size_t)world + 1);
  P.shard_tile0.resize((size_t)world + 1);
  for (int32_t r = 0; r <= world; ++r) {
    const int32_t tt = tile_b[(size_t)r];
    P.shard_row0[(size_t)r] = tt < ntiles_all ? all[(size_t)tt].row0 : (int32_t)n;
    P.shard_tile0[(size_t)r] = tt;
  }
  P.row_begin = P.shard_row0[(size_t)rank];
  P.row_end = P.shard_row0[(size_t)rank + 1];
  P.tile_begin = P.shard_tile0[(size_t)rank];
  P.tile_end = P.shard_tile0[(size_t)rank + 1];
  const int32_t nt = P.tile_end - P.tile_begin;

  // ------------------------------------------------------------ 5. layout
  // key = window<<44 | neg<<43 | local_row<<32 | internal column
  const int64_t hot_min = d->hot_min > 0 ? d->hot_min : DEFAULT_HOT_MIN;
  const uint32_t SENT_REMOTE = (uint32_t)n;  // z[n] is kept zero
  constexpr uint64_t COLM = 0x7FFFFFFFULL;
  struct TileOut {
    std::vector<Unit> units;
    std::vector<PartDesc> parts;    // chunk0 relative to the tile
    std::vector<ChunkDesc> chunks;  // ofs relative to the tile
    int32_t nhot = 0, nown = 0, nloc = 0;
    int64_t hot = 0, rem = 0, shot = 0, srem = 0, loads = 0;
  };
  std::vector<TileOut> outs((size_t)nt);
#pragma omp parallel
  {
    std::vector<uint64_t> keys, remk;
    std::vector<int32_t> rows, rb, cnt, rl;
    std::vector<uint32_t> pos;  // arranged positions of one quarter: 8 slots each
    std::vector<uint16_t> lst[8][8];
#pragma omp for schedule(dynamic, 1)
    for (int32_t lt = 0; lt < nt; ++lt) {
      const TileDesc& T = all[(size_t)(P.tile_begin + lt)];
      TileOut& O = outs[(size_t)lt];
      keys.clear();
      for (int32_t lr = 0; lr < T.nrows; ++lr) {
        const int32_t u = P.perm[(size_t)(T.row0 + lr)];
        enumerate_row(S, P.D_ptr, P.D_idx, u, [&](int32_t k, int neg) {
          const uint64_t c = (uint64_t)(uint32_t)inv[(size_t)k];
          keys.push_back(((c >> WZ_SHIFT) << 44) | ((uint64_t)neg << 43) | ((uint64_t)lr << 32) | c);
        });
      }
      std::sort(keys.begin(), keys.end());
      // one part = entries src[k0..k1) of one (window|remote, sign), sorted by (row, column)
      auto emit_part = [&](int32_t window, int32_t neg, const uint64_t* src, size_t k0, size_t k1) {
        const bool hot = window >= 0;
        PartDesc pd{window, neg, (uint32_t)O.chunks.size(), 0};
        // rows with entries, longest first
        rows.clear();
        rb.clear();
        cnt.clear();
        for (size_t k = k0; k < k1;) {
          const int32_t lr = (int32_t)((src[k] >> 32) & 0x7FF);
          size_t j = k;
          while (j < k1 && (int32_t)((src[j] >> 32) & 0x7FF) == lr) ++j;
          rows.push_back((int32_t)rows.size());
          rb.push_back((int32_t)(k - k0));
          cnt.push_back((int32_t)(j - k));
          k = j;
        }
        std::vector<int32_t> ord(rows.size());
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return cnt[(size_t)x] > cnt[(size_t)y]; });
        rl.resize(rows.size());
        for (size_t i = 0; i < rows.size(); ++i) rl[i] = (int32_t)((src[k0 + (size_t)rb[i]] >> 32) & 0x7FF);
        // ROW PIECES: few long rows -> split each row over an aligned group of lp lanes (combined by
        // a warp butterfly in the kernel) so the part still has ~16 chunks for the 16 warps
        int lp = 0;
        {
          const size_t nr = rows.size(), ne = k1 - k0;
          while (lp < 5 && nr * ((size_t)2 << lp) <= (size_t)NTHREADS && ne / (nr * ((size_t)2 << lp)) >= 16) ++lp;
        }
        // hot parts with pieces of <= 8 lanes: pack whole rows (items of 2^lp aligned lanes) into
        // residue-balanced quarters first, in the row-level numbering (ord / cnt / rb / rl by row)
        std::vector<std::array<int32_t, 32>> lanes;
        const bool pooled = hot && lp <= 3;
        if (pooled) {
          const int w = 1 << lp;
          std::vector<int32_t> lane_len(cnt.size());
          for (size_t i = 0; i < cnt.size(); ++i) lane_len[i] = (cnt[i] + w - 1) / w;  // longest piece
          std::vector<int32_t> pos_of(cnt.size());
          for (size_t p = 0; p < ord.size(); ++p) pos_of[(size_t)ord[p]] = (int32_t)p;  // row -> ord position
          plan_pools(ord, lane_len, lanes, [&](int32_t ri, int* cv) {
            for (int e = 0; e < cnt[(size_t)ri]; ++e) cv[(src[k0 + (size_t)rb[(size_t)ri] + (size_t)e] & COLM) & 7]++;
          }, w);
          if (lp > 0)  // expand items to pieces: the pieces of the row at ord position p are p*w .. p*w+w-1
            for (auto& a : lanes)
              for (int l = 0; l < 32; l += w)
                if (a[(size_t)l] >= 0) {
                  const int32_t p = pos_of[(size_t)a[(size_t)l]];
                  for (int i = 0; i < w; ++i) a[(size_t)(l + i)] = p * w + i;
                }
        }
        if (lp > 0) {
          const int pcs = 1 << lp;
          std::vector<int32_t> vrb, vcnt, vrl;
          for (int32_t ri : ord)
            for (int i = 0; i < pcs; ++i) {
              const int32_t b0 = (int32_t)((int64_t)cnt[(size_t)ri] * i / pcs);
              const int32_t b1 = (int32_t)((int64_t)cnt[(size_t)ri] * (i + 1) / pcs);
              vrb.push_back(rb[(size_t)ri] + b0);
              vcnt.push_back(b1 - b0);
              vrl.push_back(rl[(size_t)ri]);
            }
          rb.swap(vrb);
          cnt.swap(vcnt);
          rl.swap(vrl);
          ord.resize(rb.size());
          std::iota(ord.begin(), ord.end(), 0);  // units stay contiguous and lp-aligned
          pd.neg |= lp << 8;
        }
        auto slot_of = [&](int32_t ri, int e) -> uint32_t {
          return (uint32_t)((src[k0 + (size_t)rb[(size_t)ri] + (size_t)e] & COLM) - (uint64_t)window * WZ);
        };
        // chunks (lane -> row or piece); hot parts: residue-balanced quarter-warps (above)
        if (!pooled) {
          for (size_t c0 = 0; c0 < ord.size(); c0 += 32) {
            std::array<int32_t, 32> a;
            for (int l = 0; l < 32; ++l) a[(size_t)l] = c0 + (size_t)l < ord.size() ? ord[c0 + (size_t)l] : -1;
            lanes.push_back(a);
          }
        }
        for (const std::array<int32_t, 32>& lane_row : lanes) {
          ChunkDesc cd{(uint32_t)O.units.size(), 0};
          Unit hdr[HDR_UNITS];
          uint16_t* h16 = reinterpret_cast<uint16_t*>(hdr);
          for (int l = 0; l < 32; ++l)
            h16[l] = lane_row[(size_t)l] >= 0 ? (uint16_t)rl[(size_t)lane_row[(size_t)l]] : EMPTY_LANE;
          O.units.insert(O.units.end(), hdr, hdr + HDR_UNITS);
          const size_t gbase = O.units.size();
          if (hot) {
            // bank-conflict-free schedule, one quarter-warp (8 lanes) at a time
            std::vector<std::vector<uint32_t>> qpos(4);
            size_t L = 0;
            for (int q = 0; q < 4; ++q) {
              for (int l = 0; l < 8; ++l)
                for (int r = 0; r < 8; ++r) lst[l][r].clear();
              for (int l = 0; l < 8; ++l) {
                const int32_t ri = lane_row[(size_t)(q * 8 + l)];
                if (ri < 0) continue;
                for (int e = 0; e < cnt[(size_t)ri]; ++e) {
                  const uint32_t slot = slot_of(ri, e);
                  lst[l][slot & 7].push_back((uint16_t)slot);
                }
              }
              schedule_quarter(lst, qpos[(size_t)q]);
              L = std::max(L, qpos[(size_t)q].size() / 8);
            }
            // H half-groups of 4 positions: H/2 full groups of 8 slots (uint4 per lane), then one
            // trailing half-group (uint2 per lane) when H is odd
            // G full groups of 9 positions (13-bit slots packed in 16 bytes per lane), then an
            // optional tail of 4 positions (16-bit slots, 8 bytes per lane): L rounded up to 9G or 9G + 4
            uint32_t G = (uint32_t)(L / 9), tail = 0;
            const size_t rem = L - (size_t)G * 9;
            if (rem > 4) ++G;
            else if (rem > 0) tail = 1;
            cd.ng = (G << 1) | tail;
            O.units.resize(gbase + (size_t)G * 32 + tail * 16);
            auto slot_at = [&](int lane, size_t p) -> uint32_t {
              const std::vector<uint32_t>& P8 = qpos[(size_t)(lane / 8)];
              return p < P8.size() / 8 ? P8[p * 8 + (size_t)(lane & 7)] : HOT_SENT + (uint32_t)(lane & 7);
            };
            for (uint32_t g = 0; g < G; ++g)
              for (int lane = 0; lane < 32; ++lane) {
                uint64_t lo = 0, hi = 0;
                for (int e = 0; e < 9; ++e) {
                  const uint64_t v = slot_at(lane, (size_t)g * 9 + (size_t)e);
                  const int off = 13 * e;
                  if (off + 13 <= 64) lo |= v << off;
                  else if (off >= 64) hi |= v << (off - 64);
                  else {
                    lo |= v << off;
                    hi |= v >> (64 - off);
                  }
                }
                std::memcpy(O.units[gbase + (size_t)g * 32 + (size_t)lane].w, &lo, 8);
                std::memcpy(O.units[gbase + (size_t)g * 32 + (size_t)lane].w + 2, &hi, 8);
              }
            if (tail) {
              uint16_t* t16 = reinterpret_cast<uint16_t*>(O.units.data() + gbase + (size_t)G * 32);
              for (int lane = 0; lane < 32; ++lane)
                for (int e = 0; e < 4; ++e) t16[(size_t)lane * 4 + (size_t)e] = (uint16_t)slot_at(lane, (size_t)G * 9 + (size_t)e);
            }
            O.shot += (int64_t)(9 * G + 4 * tail) * 32;
          } else {
            int mx = 0;
            for (int l = 0; l < 32; ++l)
              if (lane_row[(size_t)l] >= 0) mx = std::max(mx, cnt[(size_t)lane_row[(size_t)l]]);
            const uint32_t ng = (uint32_t)((mx + 3) / 4);
            cd.ng = ng;
            O.units.resize(gbase + (size_t)ng * 32);
            for (uint32_t g = 0; g < ng; ++g)
              for (int lane = 0; lane < 32; ++lane) {
                Unit& U = O.units[gbase + (size_t)g * 32 + (size_t)lane];
                for (int e = 0; e < 4; ++e) {
                  const int p = (int)g * 4 + e;
                  uint32_t v = SENT_REMOTE;
                  const int32_t ri = lane_row[(size_t)lane];
                  // remote entries keep their sign in bit 31 (1 = complement entry, subtracted)
                  if (ri >= 0 && p < cnt[(size_t)ri]) v = (uint32_t)(src[k0 + (size_t)rb[(size_t)ri] + (size_t)p] & 0xFFFFFFFFULL);
                  U.w[e] = v;
                }
              }
            O.srem += (int64_t)ng * 128;
          }
          O.chunks.push_back(cd);
          pd.nchunks++;
        }
        O.parts.push_back(pd);
        if (hot) O.hot += (int64_t)(k1 - k0); else O.rem += (int64_t)(k1 - k0);
      };
      remk.clear();
      size_t i = 0;
      int32_t last_w = -1;
      while (i < keys.size()) {
        const uint64_t w = keys[i] >> 44;
        size_t j = i;
        while (j < keys.size() && (keys[j] >> 44) == w) ++j;
        if ((int64_t)(j - i) >= hot_min) {
          size_t m = i;  // split by sign (bit 43): non-zeros first, then complements
          while (m < j && !((keys[m] >> 43) & 1)) ++m;
          if (m > i) { emit_part((int32_t)w, 0, keys.data(), i, m); O.nhot++; }
          if (j > m) { emit_part((int32_t)w, 1, keys.data(), m, j); O.nhot++; }
          if ((int32_t)w != last_w) { O.loads++; last_w = (int32_t)w; }
        } else {  // remote: (row, sign in bit 31, column) -> one part per tile with per-entry signs
          for (size_t k = i; k < j; ++k)
            remk.push_back((keys[k] & (0x7FFULL << 32)) | (((keys[k] >> 43) & 1) << 31) | (keys[k] & COLM));
        }
        i = j;
      }
      // canonical part order (partition independent): hot windows lying wholly
      // inside the tile's own community first (always local to the rank), then the other hot
      // windows in column order, then the single remote part
      {
        const int64_t c0 = S.moff[(size_t)T.comm], c1 = S.moff[(size_t)T.comm + 1];
        auto own = [&](const PartDesc& pd) {
          return (int64_t)pd.window * WZ >= c0 && (int64_t)(pd.window + 1) * WZ <= c1;
        };
        std::stable_partition(O.parts.begin(), O.parts.end(), own);
        O.nown = (int32_t)std::count_if(O.parts.begin(), O.parts.end(), own);
        // phase A (world > 1) sums the longest prefix of those whose columns are this rank's rows
        O.nloc = 0;
        while (O.nloc < O.nown && (int64_t)O.parts[(size_t)O.nloc].window * WZ >= P.row_begin &&
               (int64_t)(O.parts[(size_t)O.nloc].window + 1) * WZ <= P.row_end)
          ++O.nloc;
      }
      if (!remk.empty()) {
        std::sort(remk.begin(), remk.end());  // (row, sign, column)
        emit_part(-1, 0, remk.data(), 0, remk.size());
      }
    }
  }
  // ------------------------------------------------------------ 6. concatenate
  P.tiles.resize((size_t)nt);
  int64_t units = 0, nparts = 0, nchunks = 0;
  for (int32_t lt = 0; lt < nt; ++lt) {
    units += (int64_t)outs[(size_t)lt].units.size();
    nparts += (int64_t)outs[(size_t)lt].parts.size();
    nchunks += (int64_t)outs[(size_t)lt].chunks.size();
  }
  if (units >= (int64_t)UINT32_MAX) { err = "index pool exceeds 64 GB"; return KUR_ERR_UNSUPPORTED; }
  P.pool.resize((size_t)std::max<int64_t>(units, 1));
  P.parts.assign((size_t)std::max<int64_t>(nparts, 1), PartDesc{-1, 0, 0, 0});
  P.chunks.assign((size_t)std::max<int64_t>(nchunks, 1), ChunkDesc{0, 0});
  int64_t uo = 0, po = 0, co = 0;
  P.n_idx_hot = P.n_idx_remote = P.n_slots_hot = P.n_slots_remote = P.n_hot_parts = P.n_window_loads = 0;
  std::vector<int64_t> uofs((size_t)nt), pofs((size_t)nt), cofs((size_t)nt);
  for (int32_t lt = 0; lt < nt; ++lt) {
    uofs[(size_t)lt] = uo;
    pofs[(size_t)lt] = po;
    cofs[(size_t)lt] = co;
    const TileOut& O = outs[(size_t)lt];
    TileDesc T = all[(size_t)(P.tile_begin + lt)];
    T.part0 = (int32_t)po;
    T.nparts = (int32_t)O.parts.size();
    T.nhot = O.nhot;
    T.nown = O.nown;
    T.nloc = O.nloc;
    P.tiles[(size_t)lt] = T;
    uo += (int64_t)O.units.size();
    po += (int64_t)O.parts.size();
    co += (int64_t)O.chunks.size();
    P.n_idx_hot += O.hot;
    P.n_idx_remote += O.rem;
    P.n_slots_hot += O.shot;
    P.n_slots_remote += O.srem;
    P.n_hot_parts += O.nhot;
    P.n_window_loads += O.loads;
  }
  // Remote parts (global z gathers, ~1 L1 wavefront each) are summed by a separate
  // k_remote pass before k_stage when they are numerous and concentrated: then the
  // latency-bound gathers get warps of their own instead of stalling a tile between
  // its shared-memory gathers.  Measured on B200 (RK stage time):
  // config 5 (42 M remote slots, 20 K per tile) 1.226 -> 1.181 ms with the pass;
  // config 4 (7.7 M, 7 K per tile) 0.312 -> 0.350 ms and config 3 (4.3 M, 17 K per
  // tile, 44 us stage) 0.044 -> 0.049 ms, so those stay inline.
  // (the count threshold applies to the whole graph -- this rank's slots x world -- so a sharded config
  // 5 keeps the pass, which at world > 1 runs on the exchange stream concurrently with phase A; the
  // per-tile threshold does not depend on the world size.  Either way the bits are the same.)
  P.split_remote = !P.small && P.n_slots_remote * world >= (16LL << 20) && nt > 0 && P.n_slots_remote / nt >= 8192;
  // World 1 with the overlapped pass (k_stage launched as k_remote's programmatic dependent, api.cpp /
  // kernels.cu, on unless KUR_REMOTE_OVERLAP=0): plans whose inline remote part would otherwise run
  // concurrently inside k_stage (small tiles, remote wavefronts >= half the hot ones: config 3) take
  // the pass instead -- config 3 29.05 K -> 29.7 K RHS/s (profiles/r02/notes/remote_overlap_pdl_ab.log).
  {
    const char* ro = std::getenv("KUR_REMOTE_OVERLAP");
    const bool overlap = world == 1 && !(ro && ro[0] == '0');
    if (overlap && !P.small && P.n_slots_remote > 0 && P.rows_per_tile <= 512 &&
        2 * P.n_slots_remote * 8 >= P.n_slots_hot)
      P.split_remote = true;
  }
  if (force_split) P.split_remote = !P.small && force_split == 1;
#pragma omp parallel for schedule(dynamic, 4)
  for (int32_t lt = 0; lt < nt; ++lt) {
    TileOut& O = outs[(size_t)lt];
    if (!O.units.empty()) std::memcpy(P.pool.data() + uofs[(size_t)lt], O.units.data(), O.units.size() * sizeof(Unit));
    for (size_t p = 0; p < O.parts.size(); ++p) {
      PartDesc pd = O.parts[p];
      pd.chunk0 += (uint32_t)cofs[(size_t)lt];
      P.parts[(size_t)pofs[(size_t)lt] + p] = pd;
    }
    for (size_t c = 0; c < O.chunks.size(); ++c) {
      ChunkDesc cd = O.chunks[c];
      cd.ofs += (uint32_t)uofs[(size_t)lt];
      P.chunks[(size_t)cofs[(size_t)lt] + c] = cd;
    }
    std::vector<Unit>().swap(O.units);
  }
  if (P.split_remote) {  // flat list of every remote chunk (one warp each in k_remote), longest first
    std::vector<std::array<uint32_t, 4>> rc;
    for (const TileDesc& T : P.tiles) {
      if (T.nparts == T.nhot) continue;
      const PartDesc& pd = P.parts[(size_t)(T.part0 + T.nhot)];
      for (uint32_t c = 0; c < pd.nchunks; ++c)
        rc.push_back({P.chunks[(size_t)(pd.chunk0 + c)].ng, pd.chunk0 + c, (uint32_t)(T.row0 - P.row_begin),
                      (uint32_t)(pd.neg >> 8)});
    }
    std::stable_sort(rc.begin(), rc.end(), [](const auto& x, const auto& y) { return x[0] > y[0]; });
    P.rchunks.resize(2 * rc.size());
    P.rem_lp.resize(rc.size());
    for (size_t k = 0; k < rc.size(); ++k) {
      P.rchunks[2 * k] = rc[k][1];
      P.rchunks[2 * k + 1] = rc[k][2];
      P.rem_lp[k] = (uint8_t)rc[k][3];
    }
  }
  // per local row: scale 1/M_m for the degree scaling (0 for a zero
  // row) and the potential constant ones_off + [z_m inside W_m]
  // (own block dense: its block sum includes z_m), see kur_potential.
  {
    const int64_t nl = P.row_end - P.row_begin;
    P.potc.assign((size_t)std::max<int64_t>(nl, 1), 0.0);
    if (d->scaling == KUR_SCALING_DEGREE) P.rowscale.assign((size_t)std::max<int64_t>(nl, 1), 0.0);
    std::vector<uint8_t> self_dense((size_t)C, 0);
    for (int32_t a = 0; a < C; ++a)
      for (int32_t i = P.D_ptr[(size_t)a]; i < P.D_ptr[(size_t)a + 1]; ++i)
        if (P.D_idx[(size_t)i] == a) self_dense[(size_t)a] = 1;
#pragma omp parallel for schedule(static)
    for (int64_t li = 0; li < nl; ++li) {
      const int32_t u = P.perm[(size_t)(P.row_begin + li)];
      P.potc[(size_t)li] = (double)ones_off[(size_t)u] + (double)self_dense[(size_t)d->community[u]];
      if (d->scaling == KUR_SCALING_DEGREE) {
        const int64_t deg = ones_off[(size_t)u] + selfl[(size_t)u];
        P.rowscale[(size_t)li] = deg > 0 ? 1.0 / (double)deg : 0.0;
      }
    }
  }
  // launch order: decreasing work (longest-processing-time first)
  P.tile_order.resize((size_t)nt);
  std::iota(P.tile_order.begin(), P.tile_order.end(), 0);
  // Launch order: longest-processing-time first per tile.  KUR_TILE_ORDER=comm (A/B): LPT at
  // community granularity (the tiles of one community adjacent, so they stage the same windows at
  // the same time -- fewer DRAM window reads, measured 0.3 % slower on config 5), =plain: tile order.
  const char* to = std::getenv("KUR_TILE_ORDER");
  if (!to || std::strcmp(to, "lpt") == 0) {
    std::stable_sort(P.tile_order.begin(), P.tile_order.end(), [&](int32_t x, int32_t y) {
      return twork[(size_t)(P.tile_begin + x)] > twork[(size_t)(P.tile_begin + y)];
    });
  } else if (std::strcmp(to, "comm") == 0) {
    std::vector<int64_t> cmax((size_t)C, 0);
    for (int32_t x = 0; x < nt; ++x) {
      const TileDesc& T = P.tiles[(size_t)x];
      cmax[(size_t)T.comm] = std::max(cmax[(size_t)T.comm], twork[(size_t)(P.tile_begin + x)]);
    }
    std::stable_sort(P.tile_order.begin(), P.tile_order.end(), [&](int32_t x, int32_t y) {
      const int32_t cx = P.tiles[(size_t)x].comm, cy = P.tiles[(size_t)y].comm;
      if (cx != cy) return cmax[(size_t)cx] != cmax[(size_t)cy] ? cmax[(size_t)cx] > cmax[(size_t)cy] : cx < cy;
      return twork[(size_t)(P.tile_begin + x)] > twork[(size_t)(P.tile_begin + y)];
    });
  }
  return KUR_OK;
}

}  // namespace kur
