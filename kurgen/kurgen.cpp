// kurgen.cpp — seeded synthetic INPUT generator shared by the oracle tests,
// the GPU parity tests and bench.py.
//
// It holds none of the method's arithmetic (no sines, no sums of phases, no
// block sums): it only draws counter-based random numbers and emits adjacency
// patterns in the row-segmented format that include/kur.h's kur_graph_desc
// describes.  Neither oracle/ nor the CUDA path includes this file; both only
// consume its outputs.
//
// RNG: SplitMix64 finaliser applied to (seed, stream, counter) — reading R18
// of DESIGN.md.  u01(seed, stream, i) is a pure function of its arguments,
// so every array is reproducible regardless of thread count.
//
// SBM sampling (reading R14): unordered pairs i<j (or the full rectangle for
// two distinct communities) are Bernoulli(p_ab), mirrored, no self-loops.
// Pairs are sampled by geometric skipping over the block's linearised pair
// set.  When p_ab > 0.5 the ZEROS are sampled instead (probability 1-p_ab)
// and the row emits a KUR_ZEROS segment for that column community.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <omp.h>

namespace {

inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

inline uint64_t bits(uint64_t seed, uint64_t stream, uint64_t i) {
  uint64_t key = mix64(seed ^ mix64(stream + 0x632BE59BD9B4E019ULL));
  return mix64(key + i * 0xD1B54A32D192ED03ULL);
}

// uniform in the open interval (0, 1)
inline double u01(uint64_t seed, uint64_t stream, uint64_t i) {
  return ((double)(bits(seed, stream, i) >> 11) + 0.5) * 0x1.0p-53;
}

struct BlockSampler {
  // enumerates sampled pairs of one unordered block pair (a <= b)
  int64_t na, nb;
  bool diag;
  double q;
  uint64_t seed, stream;
  int64_t total() const { return diag ? na * (na - 1) / 2 : na * nb; }
  template <class F> void run(F emit) const {
    const int64_t T = total();
    if (T <= 0 || q <= 0.0) return;
    int64_t i = 0, base = 0;  // diag: current row i and index of its first pair
    auto put = [&](int64_t t) {
      if (!diag) { emit(t / nb, t % nb); return; }
      while (t >= base + (na - 1 - i)) { base += na - 1 - i; ++i; }
      emit(i, i + 1 + (t - base));
    };
    if (q >= 1.0) {
      for (int64_t t = 0; t < T; ++t) put(t);
      return;
    }
    const double lq = std::log1p(-q);
    int64_t t = -1;
    uint64_t k = 0;
    for (;;) {
      double u = u01(seed, stream, k++);
      double skip = std::floor(std::log(u) / lq);
      if (skip >= (double)(T - t)) break;
      t += 1 + (int64_t)skip;
      if (t >= T) break;
      put(t);
    }
  }
};

}  // namespace

extern "C" {

// ---------------------------------------------------------------- scalars
void kg_uniform(uint64_t seed, uint64_t stream, int64_t n, double lo, double hi, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * u01(seed, stream, (uint64_t)i);
}

// Box-Muller (cosine branch), one normal per index from counters 2i, 2i+1
void kg_normal(uint64_t seed, uint64_t stream, int64_t n, double mu, double sigma, double* out) {
  const double two_pi = 6.283185307179586476925286766559;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double u1 = u01(seed, stream, 2 * (uint64_t)i);
    double u2 = u01(seed, stream, 2 * (uint64_t)i + 1);
    out[i] = mu + sigma * std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
  }
}

// standard Cauchy (location 0, scale 1) conditioned on |w| < limit by
// rejection and redraw (reading R12): attempt a of index i uses counter
// i*4096 + a.
void kg_cauchy_trunc(uint64_t seed, uint64_t stream, int64_t n, double limit, double* out) {
  const double pi = 3.14159265358979323846264338327950;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double w = 0.0;
    for (uint64_t a = 0; a < 4096; ++a) {
      double u = u01(seed, stream, (uint64_t)i * 4096 + a);
      w = std::tan(pi * (u - 0.5));
      if (std::fabs(w) < limit) break;
    }
    out[i] = w;
  }
}

// uniform random permutation (Fisher-Yates driven by the counter stream)
void kg_permutation(uint64_t seed, uint64_t stream, int64_t n, int32_t* perm) {
  for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  for (int64_t i = n - 1; i > 0; --i) {
    int64_t j = (int64_t)(bits(seed, stream, (uint64_t)i) % (uint64_t)(i + 1));
    std::swap(perm[i], perm[j]);
  }
}

// raw 64-bit draws (used by the Python side for discrete choices)
void kg_bits(uint64_t seed, uint64_t stream, int64_t n, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = bits(seed, stream, (uint64_t)i);
}

// ---------------------------------------------------------------- SBM
// Community c owns internal nodes [coff[c], coff[c+1]); perm maps an internal
// node to its user id.  P is the symmetric C x C edge-probability matrix.
// edge stream of unordered block pair (a<=b): stream_base + a*C + b.
//
// Pass 1: per-user-row stored-entry counts (row_cnt[n], zero-initialised by
// the caller) — returns the total.
int64_t kg_sbm_count(int64_t n, int32_t C, const int64_t* coff, const double* P,
                     const int32_t* perm, uint64_t seed, uint64_t stream_base,
                     int64_t* row_cnt) {
  (void)n;
  std::atomic<int64_t> total{0};
  const int64_t npairs = (int64_t)C * (C + 1) / 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t pi = 0; pi < npairs; ++pi) {
    // decode pi -> (a, b) with a <= b (row-major over a)
    int64_t a = 0, rem = pi;
    while (rem >= C - a) { rem -= C - a; ++a; }
    int64_t b = a + rem;
    double p = P[a * C + b];
    BlockSampler s{coff[a + 1] - coff[a], coff[b + 1] - coff[b], a == b,
                   p > 0.5 ? 1.0 - p : p, seed, stream_base + (uint64_t)(a * C + b)};
    int64_t local = 0;
    const int64_t oa = coff[a], ob = coff[b];
    s.run([&](int64_t i, int64_t j) {
      int32_t ua = perm[oa + i], ub = perm[ob + j];
      __atomic_fetch_add(&row_cnt[ua], 1, __ATOMIC_RELAXED);
      __atomic_fetch_add(&row_cnt[ub], 1, __ATOMIC_RELAXED);
      local += 2;
    });
    total += local;
  }
  return total.load();
}

// Pass 2: fill cols (user column ids) at row_ptr[u] + atomic cursor, then sort
// every row by (label(col), col).  row_fill[n] is scratch (zeroed here).
void kg_sbm_fill(int64_t n, int32_t C, const int64_t* coff, const double* P,
                 const int32_t* perm, const int32_t* labels, uint64_t seed,
                 uint64_t stream_base, const int64_t* row_ptr, int32_t* cols,
                 int64_t* row_fill) {
  std::memset(row_fill, 0, sizeof(int64_t) * (size_t)n);
  const int64_t npairs = (int64_t)C * (C + 1) / 2;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t pi = 0; pi < npairs; ++pi) {
    int64_t a = 0, rem = pi;
    while (rem >= C - a) { rem -= C - a; ++a; }
    int64_t b = a + rem;
    double p = P[a * C + b];
    BlockSampler s{coff[a + 1] - coff[a], coff[b + 1] - coff[b], a == b,
                   p > 0.5 ? 1.0 - p : p, seed, stream_base + (uint64_t)(a * C + b)};
    const int64_t oa = coff[a], ob = coff[b];
    s.run([&](int64_t i, int64_t j) {
      int32_t ua = perm[oa + i], ub = perm[ob + j];
      int64_t pa = __atomic_fetch_add(&row_fill[ua], 1, __ATOMIC_RELAXED);
      int64_t pb = __atomic_fetch_add(&row_fill[ub], 1, __ATOMIC_RELAXED);
      cols[row_ptr[ua] + pa] = ub;
      cols[row_ptr[ub] + pb] = ua;
    });
  }
#pragma omp parallel
  {
    std::vector<uint64_t> key;
#pragma omp for schedule(dynamic, 256)
    for (int64_t u = 0; u < n; ++u) {
      int64_t b0 = row_ptr[u], b1 = row_ptr[u + 1];
      key.resize((size_t)(b1 - b0));
      for (int64_t e = b0; e < b1; ++e)
        key[(size_t)(e - b0)] = ((uint64_t)(uint32_t)labels[cols[e]] << 32) | (uint32_t)cols[e];
      std::sort(key.begin(), key.end());
      for (int64_t e = b0; e < b1; ++e) cols[e] = (int32_t)(uint32_t)key[(size_t)(e - b0)];
    }
  }
}

// Pass 3: segments.  Row u (community a = labels[u]) gets, in increasing
// column-community order b: a KUR_ZEROS segment for every b with P[a][b] > 0.5
// (possibly empty), and a KUR_ONES segment for every other b with entries.
// With seg_ptr == NULL only seg_cnt[n] is written; returns total segments.
int64_t kg_sbm_segments(int64_t n, int32_t C, const int32_t* labels, const double* P,
                        const int64_t* row_ptr, const int32_t* cols, int64_t* seg_cnt,
                        const int64_t* seg_ptr, int32_t* seg_comm, uint8_t* seg_kind,
                        int64_t* idx_ptr) {
  // dense (ZEROS-mode) partner lists per community
  std::vector<std::vector<int32_t>> zmode((size_t)C);
  for (int32_t a = 0; a < C; ++a)
    for (int32_t b = 0; b < C; ++b)
      if (P[(int64_t)a * C + b] > 0.5) zmode[(size_t)a].push_back(b);
  std::atomic<int64_t> total{0};
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t u = 0; u < n; ++u) {
    const int32_t a = labels[u];
    const std::vector<int32_t>& zm = zmode[(size_t)a];
    int64_t e = row_ptr[u], e1 = row_ptr[u + 1];
    size_t zi = 0;
    int64_t ns = 0;
    int64_t s = seg_ptr ? seg_ptr[u] : 0;
    auto emit = [&](int32_t b, uint8_t kind, int64_t from, int64_t to) {
      if (seg_ptr) {
        seg_comm[s] = b;
        seg_kind[s] = kind;
        idx_ptr[s] = from;
        (void)to;
        ++s;
      }
      ++ns;
    };
    while (e < e1 || zi < zm.size()) {
      int32_t be = e < e1 ? labels[cols[e]] : C;
      int32_t bz = zi < zm.size() ? zm[zi] : C;
      int32_t b = std::min(be, bz);
      int64_t f = e;
      while (f < e1 && labels[cols[f]] == b) ++f;
      emit(b, bz == b ? 1 : 0, e, f);
      if (bz == b) ++zi;
      e = f;
    }
    seg_cnt[u] = ns;
    total += ns;
  }
  return total.load();
}

}  // extern "C"
