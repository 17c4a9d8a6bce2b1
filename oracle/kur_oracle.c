/* kur_oracle.c — the CPU ORACLE for the Kuramoto-on-graphs hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load, call or link this
 * file.  It shares no code, header, table or constant generator with the CUDA
 * path (paper_2102_07167_b200/): the graph arrays it reads are the seeded
 * inputs kurgen/ produces, in the row-segmented layout whose meaning is
 * re-declared below independently of include/kur.h.
 *
 * What it computes is the PLAIN DEFINITION of the right-hand side of the
 * Kuramoto model on a graph with uniform scaling (eq.
 * KuramotoGraph, with the scaling M_m = M of P:404-408):
 *
 *     theta_m' = omega_m + (K/M) * sum_l A_ml sin(theta_l - theta_m)
 *
 * evaluated by direct O(nnz) summation — no block sums, no localised order
 * parameters, no permutation.  The community labels are
 * used ONLY to decode KUR_ZEROS segments into the explicit list of ones.
 * orc_graph_set_scaling selects the non-uniform scaling M_m = sum_l A_ml of
 * P:409-415 instead (zero rows: theta_m' = omega_m),
 * and orc_potential evaluates the potential V of P:474-487 (NEXT-1).
 *
 * Three evaluation modes:
 *   ORC_NAIVE  (0)  per-edge sin(theta_l - theta_m), P:388 (and P:130 for the
 *                   complete graph);
 *   ORC_MATVEC (1)  the componentwise-product form of P:443-444,
 *                   G = omega + K((Asin).*cos - (Acos).*sin), A = A/M, with the
 *                   same row enumeration (still O(nnz), no block sums);
 *   ORC_OP     (2)  the order-parameter form of P:249-255,
 *                   theta' = omega + K r sin(psi - theta) — valid for the
 *                   complete graph only (the diagonal term sin(0)=0 is
 *                   "neglected").
 * Time stepping: classical RK4 with fixed step h (reading R8 of DESIGN.md),
 * stages in the order theta(1)=theta_n, theta(2)=theta_n+(h/2)k1,
 * theta(3)=theta_n+(h/2)k2, theta(4)=theta_n+h k3,
 * theta_{n+1}=theta_n+(h/6)(k1+2k2+2k3+k4) (P:297-321,
 * P:374).  The state is never wrapped (reading R9).
 * Order parameter: r e^{i psi} = (1/M) sum_m e^{i theta_m} = C_M + i S_M
 * (P:236-239), r = sqrt(C^2+S^2), psi = atan2(S, C), psi = 0 when r = 0
 * (reading R11).
 *
 * Arithmetic: IEEE double, compiled -O2 -fno-fast-math -ffp-contract=off;
 * every per-row sum is sequential in enumeration order, so results are
 * identical for any OpenMP thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

enum { ORC_NAIVE = 0, ORC_MATVEC = 1, ORC_OP = 2, ORC_COSINE = 3 /* internal: potential */ };
enum { SEG_ONES = 0, SEG_ZEROS = 1 }; /* row-segment kinds (see kurgen/) */

/* Graph as given by the caller (user numbering):
 *   row u owns segments seg_ptr[u] .. seg_ptr[u+1]-1;
 *   segment s covers column community seg_comm[s]; its list is
 *   idx[idx_ptr[s] .. idx_ptr[s+1]-1] (ascending user ids inside that
 *   community);  kind ONES: listed columns are the ones of row u in that
 *   community; kind ZEROS: listed columns are the zeros, every other member
 *   of the community is a one.  Communities without a segment are zero.
 *   The diagonal l == m never contributes. */
typedef struct {
  int64_t n;
  int32_t n_comm;
  const int32_t *community;
  const int64_t *seg_ptr;
  const int32_t *seg_comm;
  const uint8_t *seg_kind;
  const int64_t *idx_ptr;
  const int32_t *idx;
  int64_t *member_off; /* [n_comm+1] */
  int32_t *members;    /* ascending user ids per community */
  int scaling;         /* ORC_UNIFORM: M_m = M; ORC_DEGREE: M_m = sum_l A_ml */
} orc_graph;

enum { ORC_UNIFORM = 0, ORC_DEGREE = 1 };

/* Select the scaling M_m of P:388 (reading R22 of DESIGN.md for the degree:
 * the off-diagonal ones plus A_mm, which is 1 only when m is listed in a
 * KUR_ONES segment of its own community). */
void orc_graph_set_scaling(orc_graph *g, int scaling) { g->scaling = scaling; }

/* 1 iff row u lists itself in a ONES segment (a stored self-loop). */
static int self_loop(const orc_graph *g, int64_t u) {
  for (int64_t sg = g->seg_ptr[u]; sg < g->seg_ptr[u + 1]; ++sg) {
    if (g->seg_kind[sg] != SEG_ONES || g->seg_comm[sg] != g->community[u]) continue;
    for (int64_t e = g->idx_ptr[sg]; e < g->idx_ptr[sg + 1]; ++e)
      if (g->idx[e] == u) return 1;
  }
  return 0;
}

orc_graph *orc_graph_new(int64_t n, int32_t n_comm, const int32_t *community,
                         const int64_t *seg_ptr, const int32_t *seg_comm,
                         const uint8_t *seg_kind, const int64_t *idx_ptr,
                         const int32_t *idx) {
  orc_graph *g = (orc_graph *)calloc(1, sizeof(orc_graph));
  g->n = n;
  g->n_comm = n_comm;
  g->community = community;
  g->seg_ptr = seg_ptr;
  g->seg_comm = seg_comm;
  g->seg_kind = seg_kind;
  g->idx_ptr = idx_ptr;
  g->idx = idx;
  g->member_off = (int64_t *)calloc((size_t)n_comm + 1, sizeof(int64_t));
  g->members = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t u = 0; u < n; ++u) g->member_off[community[u] + 1]++;
  for (int32_t c = 0; c < n_comm; ++c) g->member_off[c + 1] += g->member_off[c];
  int64_t *fill = (int64_t *)calloc((size_t)n_comm + 1, sizeof(int64_t));
  for (int64_t u = 0; u < n; ++u) { /* ascending u => ascending members */
    int32_t c = community[u];
    g->members[g->member_off[c] + fill[c]++] = (int32_t)u;
  }
  free(fill);
  return g;
}

void orc_graph_free(orc_graph *g) {
  if (!g) return;
  free(g->member_off);
  free(g->members);
  free(g);
}

/* Visit the columns l with A_ul = 1, l != u, in segment order (ascending
 * within a segment).  Returns the number visited.  mode NAIVE accumulates
 * sin(theta_l - theta_u) into *a0; mode MATVEC accumulates sin(theta_l) into
 * *a0 and cos(theta_l) into *a1 (from the precomputed tables s, c). */
static int64_t row_sums(const orc_graph *g, int64_t u, int mode, const double *theta,
                        const double *s, const double *c, double *a0, double *a1) {
  double acc0 = 0.0, acc1 = 0.0;
  int64_t cnt = 0;
  const double tu = theta[u];
#define ORC_TERM(l)                                   \
  do {                                                \
    if ((l) != u) {                                   \
      if (mode == ORC_NAIVE) {                        \
        acc0 += sin(theta[(l)] - tu);                 \
      } else if (mode == ORC_COSINE) {                \
        acc0 += cos(theta[(l)] - tu);                 \
      } else {                                        \
        acc0 += s[(l)];                               \
        acc1 += c[(l)];                               \
      }                                               \
      ++cnt;                                          \
    }                                                 \
  } while (0)
  for (int64_t sg = g->seg_ptr[u]; sg < g->seg_ptr[u + 1]; ++sg) {
    const int32_t *lst = g->idx + g->idx_ptr[sg];
    const int64_t len = g->idx_ptr[sg + 1] - g->idx_ptr[sg];
    if (g->seg_kind[sg] == SEG_ONES) {
      for (int64_t e = 0; e < len; ++e) ORC_TERM((int64_t)lst[e]);
    } else { /* members of the community minus the listed zeros (merge walk) */
      const int32_t b = g->seg_comm[sg];
      const int32_t *mem = g->members + g->member_off[b];
      const int64_t nm = g->member_off[b + 1] - g->member_off[b];
      int64_t z = 0;
      for (int64_t e = 0; e < nm; ++e) {
        const int32_t l = mem[e];
        while (z < len && lst[z] < l) ++z;
        if (z < len && lst[z] == l) continue;
        ORC_TERM((int64_t)l);
      }
    }
  }
#undef ORC_TERM
  *a0 = acc0;
  *a1 = acc1;
  return cnt;
}

/* (1/M) sum cos, (1/M) sum sin — P:158-159 / P:238, sequential. */
static void order_sums(int64_t n, const double *theta, double *C, double *S) {
  double sc = 0.0, ss = 0.0;
  for (int64_t m = 0; m < n; ++m) {
    sc += cos(theta[m]);
    ss += sin(theta[m]);
  }
  *C = sc / (double)n;
  *S = ss / (double)n;
}

/* r and psi of the complex order parameter (reading R11). */
void orc_order_parameter(int64_t n, const double *theta, double *r_psi) {
  double C, S;
  order_sums(n, theta, &C, &S);
  double r = sqrt(C * C + S * S);
  r_psi[0] = r;
  r_psi[1] = (r == 0.0) ? 0.0 : atan2(S, C);
}

/* Right-hand side for the rows listed in `rows` (user ids; NULL = all rows,
 * out[u]); with rows != NULL, out[i] is the value of row rows[i].
 * Returns 0 on success, -1 on a bad mode. */
int orc_rhs(const orc_graph *g, int mode, double K, const double *theta,
            const double *omega, int64_t nrows, const int64_t *rows, double *out) {
  const int64_t n = g->n;
  if (mode != ORC_NAIVE && mode != ORC_MATVEC && mode != ORC_OP) return -1;
  const int64_t cnt = rows ? nrows : n;
  if (mode == ORC_OP && g->scaling != ORC_UNIFORM) return -1; /* classical model only */
  if (mode == ORC_OP) {
    double C, S;
    order_sums(n, theta, &C, &S);
    const double r = sqrt(C * C + S * S);
    const double psi = (r == 0.0) ? 0.0 : atan2(S, C);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
      const int64_t m = rows ? rows[i] : i;
      out[i] = omega[m] + K * r * sin(psi - theta[m]);
    }
    return 0;
  }
  double *s = NULL, *c = NULL;
  if (mode == ORC_MATVEC) { /* sin(theta), cos(theta) once ("2M") */
    s = (double *)malloc(sizeof(double) * (size_t)n);
    c = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < n; ++l) {
      s[l] = sin(theta[l]);
      c[l] = cos(theta[l]);
    }
  }
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < cnt; ++i) {
    const int64_t m = rows ? rows[i] : i;
    double a0, a1;
    const int64_t ones = row_sums(g, m, mode, theta, s, c, &a0, &a1);
    /* scaling M_m: uniform M or the row degree */
    const double M = g->scaling == ORC_UNIFORM ? (double)n : (double)(ones + self_loop(g, m));
    if (M == 0.0) { /* zero row: theta_m' = omega_m, "the scaling is dispensible" */
      out[i] = omega[m];
      continue;
    }
    if (mode == ORC_NAIVE) {
      out[i] = omega[m] + (K / M) * a0;
    } else {
      const double As = a0 / M, Ac = a1 / M; /* (A sin)_m, (A cos)_m with A = A/M_m */
      out[i] = omega[m] + K * (As * c[m] - Ac * s[m]);
    }
  }
  free(s);
  free(c);
  return 0;
}

/* Number of ones per row (diagonal excluded) — used by tests and by the
 * cost counters. */
void orc_row_degree(const orc_graph *g, int64_t *deg) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t u = 0; u < g->n; ++u) {
    int64_t cnt = 0;
    for (int64_t sg = g->seg_ptr[u]; sg < g->seg_ptr[u + 1]; ++sg) {
      const int64_t len = g->idx_ptr[sg + 1] - g->idx_ptr[sg];
      const int32_t *lst = g->idx + g->idx_ptr[sg];
      int diag_listed = 0;
      for (int64_t e = 0; e < len; ++e) diag_listed |= (lst[e] == u);
      if (g->seg_kind[sg] == SEG_ONES) {
        cnt += len - diag_listed;
      } else {
        const int32_t b = g->seg_comm[sg];
        const int64_t nm = g->member_off[b + 1] - g->member_off[b];
        const int in_b = (g->community[u] == b);
        cnt += nm - len - (in_b && !diag_listed ? 1 : 0);
      }
    }
    deg[u] = cnt;
  }
}

/* Classical RK4 with fixed step h, nsteps steps, theta in/out (user order).
 * r_trace (may be NULL): (r, psi) of theta_n for n = 0, re, 2re, ... <= nsteps,
 * i.e. floor(nsteps/re)+1 pairs; record_every <= 0 disables recording.
 * theta10 (may be NULL): copy of theta after min(10, nsteps) steps. */
int orc_rk4(const orc_graph *g, int mode, double K, double h, int64_t nsteps,
            int32_t record_every, double *theta, const double *omega, double *r_trace,
            double *theta10) {
  const int64_t n = g->n;
  double *k1 = (double *)malloc(sizeof(double) * (size_t)n);
  double *k2 = (double *)malloc(sizeof(double) * (size_t)n);
  double *k3 = (double *)malloc(sizeof(double) * (size_t)n);
  double *k4 = (double *)malloc(sizeof(double) * (size_t)n);
  double *ts = (double *)malloc(sizeof(double) * (size_t)n);
  int rc = 0;
  for (int64_t step = 0; step <= nsteps; ++step) {
    if (r_trace && record_every > 0 && step % record_every == 0)
      orc_order_parameter(n, theta, r_trace + 2 * (step / record_every));
    if (theta10 && step == (nsteps < 10 ? nsteps : 10))
      memcpy(theta10, theta, sizeof(double) * (size_t)n);
    if (step == nsteps) break;
    if ((rc = orc_rhs(g, mode, K, theta, omega, 0, NULL, k1))) break;
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < n; ++m) ts[m] = theta[m] + (h / 2.0) * k1[m];
    orc_rhs(g, mode, K, ts, omega, 0, NULL, k2);
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < n; ++m) ts[m] = theta[m] + (h / 2.0) * k2[m];
    orc_rhs(g, mode, K, ts, omega, 0, NULL, k3);
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < n; ++m) ts[m] = theta[m] + h * k3[m];
    orc_rhs(g, mode, K, ts, omega, 0, NULL, k4);
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < n; ++m)
      theta[m] = theta[m] + (h / 6.0) * (k1[m] + 2.0 * k2[m] + 2.0 * k3[m] + k4[m]);
  }
  free(k1);
  free(k2);
  free(k3);
  free(k4);
  free(ts);
  return rc;
}

/* Other one-step integrators of the paper, fixed step h:
 *   ORC_EULER (1): theta_{n+1} = theta_n + h F(theta_n)
 *   ORC_HEUN  (2): k1 = F(theta_n), k2 = F(theta_n + h k1),
 *                  theta_{n+1} = theta_n + (h/2)(k1 + k2)           (2nd-order explicit RK)
 *   ORC_IMPMID(3): theta_{n+1} = theta_n + h F((theta_n + theta_{n+1})/2), solved by fixed-point
 *                  iteration from the Euler predictor until max|update| <= fp_tol or fp_max_iter
 *                  iterations (2nd-order implicit, geometric; reading R23)
 * (method 0 = classical RK4 is orc_rk4).  r_trace as in orc_rk4.  Returns 0, -1 on a bad method. */
int orc_step_method(const orc_graph *g, int method, int mode, double K, double h, int64_t nsteps,
                    int32_t record_every, double *theta, const double *omega, double *r_trace,
                    double fp_tol, int32_t fp_max_iter) {
  if (method < 1 || method > 3) return -1;
  const int64_t n = g->n;
  double *k1 = (double *)malloc(sizeof(double) * (size_t)n);
  double *k2 = (double *)malloc(sizeof(double) * (size_t)n);
  double *ts = (double *)malloc(sizeof(double) * (size_t)n);
  double *tp = (double *)malloc(sizeof(double) * (size_t)n);
  for (int64_t step = 0; step <= nsteps; ++step) {
    if (r_trace && record_every > 0 && step % record_every == 0)
      orc_order_parameter(n, theta, r_trace + 2 * (step / record_every));
    if (step == nsteps) break;
    orc_rhs(g, mode, K, theta, omega, 0, NULL, k1);
    if (method == 1) {
      for (int64_t m = 0; m < n; ++m) theta[m] = theta[m] + h * k1[m];
    } else if (method == 2) {
      for (int64_t m = 0; m < n; ++m) ts[m] = theta[m] + h * k1[m];
      orc_rhs(g, mode, K, ts, omega, 0, NULL, k2);
      for (int64_t m = 0; m < n; ++m) theta[m] = theta[m] + (h / 2.0) * (k1[m] + k2[m]);
    } else {
      for (int64_t m = 0; m < n; ++m) tp[m] = theta[m] + h * k1[m]; /* Euler predictor */
      for (int32_t it = 0; it < fp_max_iter; ++it) {
        for (int64_t m = 0; m < n; ++m) ts[m] = (theta[m] + tp[m]) / 2.0;
        orc_rhs(g, mode, K, ts, omega, 0, NULL, k2);
        double diff = 0.0;
        for (int64_t m = 0; m < n; ++m) {
          const double nv = theta[m] + h * k2[m];
          const double d = fabs(nv - tp[m]);
          if (d > diff) diff = d;
          tp[m] = nv;
        }
        if (diff <= fp_tol) break;
      }
      memcpy(theta, tp, sizeof(double) * (size_t)n);
    }
  }
  free(k1);
  free(k2);
  free(ts);
  free(tp);
  return 0;
}

/* Variable-step classical RK4 ("a variable stepsize fourth-order explicit
 * Runge-Kutta method"; the controller is unstated, reading R25 follows
 * SPEC S:309): from (t = 0, theta) to t_end.  Each trial step of size
 * h (h = t_end - t for the last step, i.e. when t + h >= t_end - 1e-12 h) computes y1 = one RK4 step of h and y2 = two RK4 steps
 * of h/2 (step doubling), the error
 *     err = sqrt( (1/N) sum_m ((y2_m - y1_m) / (atol + rtol |y2_m|))^2 ) / 15
 * (the sum sequential in m), accepts iff err <= 1 (theta = y2, t += h), and sets
 *     h <- clamp(h * min(fac_max, max(fac_min, safety * err^(-1/5))), h_min, h_max)
 * (factor fac_max when err = 0).  Accepted (t, h, r, psi) are written to the
 * out arrays (capacity cap).  Returns the number of accepted steps, -1 if a
 * rejected step had h <= h_min, -2 on a non-finite error, -3 when max_trials
 * trials did not reach t_end. */
int64_t orc_integrate_adaptive(const orc_graph *g, int mode, double K, double t_end, double h0, double h_min,
                               double h_max, double atol, double rtol, double safety, double fac_min, double fac_max,
                               int64_t max_trials, double *theta, const double *omega, int64_t cap, double *t_out,
                               double *h_out, double *rpsi_out, int64_t *n_rejected) {
  const int64_t n = g->n;
  double *y1 = (double *)malloc(sizeof(double) * (size_t)n);
  double *y2 = (double *)malloc(sizeof(double) * (size_t)n);
  double t = 0.0, h = h0;
  int64_t acc = 0, rej = 0, trials = 0, rc = 0;
  while (t < t_end) {
    if (trials++ >= max_trials) { rc = -3; break; }
    /* the last step lands exactly on t_end (also when t + h misses it by rounding only) */
    const int last = !(t + h < t_end - 1e-12 * h);
    const double hs = last ? t_end - t : h;
    memcpy(y1, theta, sizeof(double) * (size_t)n);
    orc_rk4(g, mode, K, hs, 1, 0, y1, omega, NULL, NULL);
    memcpy(y2, theta, sizeof(double) * (size_t)n);
    orc_rk4(g, mode, K, hs / 2.0, 2, 0, y2, omega, NULL, NULL);
    double ss = 0.0;
    for (int64_t m = 0; m < n; ++m) {
      const double e = (y2[m] - y1[m]) / (atol + rtol * fabs(y2[m]));
      ss += e * e;
    }
    const double err = sqrt(ss / (double)n) / 15.0;
    if (!isfinite(err)) { rc = -2; break; }
    if (err <= 1.0) {
      memcpy(theta, y2, sizeof(double) * (size_t)n);
      t = last ? t_end : t + hs;
      if (acc < cap) {
        if (t_out) t_out[acc] = t;
        if (h_out) h_out[acc] = hs;
        if (rpsi_out) orc_order_parameter(n, theta, rpsi_out + 2 * acc);
      }
      ++acc;
    } else {
      ++rej;
      if (hs <= h_min) { rc = -1; break; }
    }
    double fac = err == 0.0 ? fac_max : safety * pow(err, -0.2);
    if (fac > fac_max) fac = fac_max;
    if (fac < fac_min) fac = fac_min;
    h = hs * fac;
    if (h > h_max) h = h_max;
    if (h < h_min) h = h_min;
  }
  if (n_rejected) *n_rejected = rej;
  free(y1);
  free(y2);
  return rc ? rc : acc;
}

/* Potential of the model on a graph (eq. ExtendedPotentialConservation;
 * P:221-233 for the complete graph), evaluated from its definition
 *     V = -sum_m omega_m theta_m + (K/2) sum_{m,l} (A_ml / M_m) (1 - cos(theta_l - theta_m)),
 * with M_m the graph's scaling (rows with M_m = 0 contribute nothing).  Per-row
 * terms are computed in parallel, then summed sequentially in row order. */
double orc_potential(const orc_graph *g, double K, const double *theta, const double *omega) {
  const int64_t n = g->n;
  double *term = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t m = 0; m < n; ++m) {
    double a0, a1;
    const int64_t ones = row_sums(g, m, ORC_COSINE, theta, NULL, NULL, &a0, &a1);
    const double M = g->scaling == ORC_UNIFORM ? (double)n : (double)(ones + self_loop(g, m));
    term[m] = M == 0.0 ? 0.0 : ((double)ones - a0) / M; /* sum_l A_ml (1 - cos), diagonal term 0 */
  }
  double wt = 0.0, s = 0.0;
  for (int64_t m = 0; m < n; ++m) {
    wt += omega[m] * theta[m];
    s += term[m];
  }
  free(term);
  return -wt + (K / 2.0) * s;
}

int orc_num_threads(void) { return omp_get_max_threads(); }
void orc_set_num_threads(int t) { omp_set_num_threads(t); }
