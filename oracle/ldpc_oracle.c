/*
 * ldpc_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C, float64 restatement of the reference's numba engine
 * (/root/reference/pkg/src/ldpc_ids/_engine.py, cited below as E:<line>).
 * It is the checker for the CUDA decoder in paper_2102_11089_b200/csrc and
 * the CPU-baseline arm of bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the product
 * decode path never does.
 *
 * Parity pin: the eight reference schedules are checked bit-for-bit against
 * golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py writes tests/golden/NAME.npz; tests/test_oracle.py).
 * Operation order follows the reference exactly (sequential tanh products,
 * sequential sums in vn_edges order, same libm calls), built with
 * -ffp-contract=off so no FMA contraction changes a rounding.
 *
 * The two schedules the reference does not have (SURVEY.md sec.8(a) rows
 * a20/a21) are DEFINED here and are "parity unpinned" by the reference:
 *   KIND_LAYERED : row-layered BP, checks m = 0..M-1 in order; for each check
 *                  v2c = clamp(total - c2v) over N(m), c2v' = cn_msg(v2c),
 *                  total += c2v' - c2v (the E:147 incremental form).
 *                  Trace rows (want_trace): pre_total = chl + sum of the
 *                  C2V messages a flooding pass would send from the current
 *                  extrinsics v2c = clamp(total - c2v) (E:768-782 semantics).
 *   KIND_ME_RBP  : multi-edge RBP; per round the n_p largest residuals
 *                  (ties -> lowest edge id) are propagated in ascending edge
 *                  id, each committing its then-current pre_c2v.  Boundaries
 *                  as E:633-642.  n_p = 1 reproduces _decode_rbp exactly.
 *
 * Build: see oracle/Makefile (REAL=double is the oracle; REAL=float builds a
 * diagnostic single-precision variant used only to estimate fp32 drift).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#ifndef OR_REAL
#define OR_REAL double
#endif
typedef OR_REAL real;

#ifdef OR_SINGLE
#define R_TANH tanhf
#define R_ATANH atanhf
#define R_EXP expf
#define R_ABS fabsf
#else
#define R_TANH tanh
#define R_ATANH atanh
#define R_EXP exp
#define R_ABS fabs
#endif

#define LLR_MAX ((real)30.0)                 /* E:13 */
#define ATANH_CLIP ((real)(1.0 - 1e-12))     /* E:14 */

enum { C_PROP = 0, C_V2C, C_PRE, C_CI, C_CMP, C_MSEL, C_KHITS, C_KTRIALS, N_COUNTERS }; /* E:17-25 */
enum { KERNEL_EXACT = 0, KERNEL_MINSUM = 1 };                                          /* E:27-28 */
enum {
  KIND_FLOODING = 0, KIND_RBP = 1, KIND_CIRBP = 2, KIND_LMDRBP = 3, KIND_SLMDRBP = 4,
  KIND_LMD_CIRBP = 5, KIND_ME_CIRBP = 6, KIND_ME_LMD_CIRBP = 7, KIND_LAYERED = 8, KIND_ME_RBP = 9
};

typedef struct {
  int64_t n_vars, n_checks, n_edges;
  const int64_t *edge_cn, *edge_vn, *cn_ptr, *vn_ptr, *vn_edges;
} graph_t;

typedef struct {
  int kind, kernel, i_max, n_p, n_g;
  int64_t k_info;
  double gamma;
  int64_t seed;
} sched_t;

/* per-update log used by the near-tie analysis (tests only) */
typedef struct {
  int64_t cap, len;
  int64_t* edge;   /* propagated edge id */
  double* c2v;     /* committed C2V value */
  double* gap;     /* smallest relative top-2 gap among the selections made for this update */
} steplog_t;

typedef struct {
  real *c2v, *v2c, *pre, *res, *total, *pre_total, *ci, *th;
  int64_t* counters;
  int64_t *biterr, *biterr_info;
  double* trace;   /* (i_max+1) x 2N or NULL */
  steplog_t* log;
  double cur_gap;
} state_t;

/* ---------------------------------------------------------------- helpers */

static inline real clampv(real x) {   /* E:31-37 */
  if (x > LLR_MAX) return LLR_MAX;
  if (x < -LLR_MAX) return -LLR_MAX;
  return x;
}

static inline real p0(real llr) {     /* E:40-46 */
  if (llr >= (real)0.0) return (real)1.0 / ((real)1.0 + R_EXP(-llr));
  real e = R_EXP(llr);
  return e / ((real)1.0 + e);
}

static inline real ci_of(real t, real pt) { return R_ABS(p0(t) - p0(pt)); }

/* E:49-82 */
static real cn_msg(const real* v2c, const graph_t* g, int64_t m, int64_t skip, int kernel) {
  if (kernel == KERNEL_EXACT) {
    real prod = 1.0;
    int64_t count = 0;
    for (int64_t e = g->cn_ptr[m]; e < g->cn_ptr[m + 1]; ++e) {
      if (e == skip) continue;
      prod *= R_TANH((real)0.5 * clampv(v2c[e]));
      count++;
    }
    if (count == 0) return 0.0;
    if (prod > ATANH_CLIP) prod = ATANH_CLIP;
    else if (prod < -ATANH_CLIP) prod = -ATANH_CLIP;
    return clampv((real)2.0 * R_ATANH(prod));
  }
  real sign = 1.0, mag = (real)1e30;
#ifndef OR_SINGLE
  mag = 1e300;
#endif
  int64_t count = 0;
  for (int64_t e = g->cn_ptr[m]; e < g->cn_ptr[m + 1]; ++e) {
    if (e == skip) continue;
    real v = clampv(v2c[e]);
    if (v < (real)0.0) { sign = -sign; v = -v; }
    if (v < mag) mag = v;
    count++;
  }
  if (count == 0) return 0.0;
  return clampv(sign * mag);
}

/* E:85-103 */
static real cn_msg_cached(const real* th, const real* v2c, const graph_t* g, int64_t m,
                          int64_t skip, int kernel) {
  if (kernel != KERNEL_EXACT) return cn_msg(v2c, g, m, skip, kernel);
  real prod = 1.0;
  int64_t count = 0;
  for (int64_t e = g->cn_ptr[m]; e < g->cn_ptr[m + 1]; ++e) {
    if (e == skip) continue;
    prod *= th[e];
    count++;
  }
  if (count == 0) return 0.0;
  if (prod > ATANH_CLIP) prod = ATANH_CLIP;
  else if (prod < -ATANH_CLIP) prod = -ATANH_CLIP;
  return clampv((real)2.0 * R_ATANH(prod));
}

/* E:106-127 */
static void init_state(const real* chl, const graph_t* g, int kernel, state_t* s) {
  for (int64_t e = 0; e < g->n_edges; ++e) {
    s->c2v[e] = 0.0;
    s->v2c[e] = clampv(chl[g->edge_vn[e]]);
    s->th[e] = R_TANH((real)0.5 * s->v2c[e]);
  }
  for (int64_t n = 0; n < g->n_vars; ++n) s->total[n] = chl[n];
  for (int64_t m = 0; m < g->n_checks; ++m)
    for (int64_t e = g->cn_ptr[m]; e < g->cn_ptr[m + 1]; ++e) {
      s->pre[e] = cn_msg(s->v2c, g, m, e, kernel);
      s->res[e] = R_ABS(s->pre[e] - s->c2v[e]);
    }
  for (int64_t n = 0; n < g->n_vars; ++n) {
    real acc = chl[n];
    for (int64_t k = g->vn_ptr[n]; k < g->vn_ptr[n + 1]; ++k) acc += s->pre[g->vn_edges[k]];
    s->pre_total[n] = acc;
    s->ci[n] = ci_of(s->total[n], s->pre_total[n]);
  }
}

/* ------------------------------------------------- max tree (E:220-257) */

typedef struct { real* t; int64_t size; } tree_t;

static void tree_build(tree_t* tr, const real* v, int64_t n) {
  int64_t size = 1;
  while (size < n) size *= 2;
  tr->size = size;
  tr->t = (real*)malloc(sizeof(real) * 2 * size);
  for (int64_t i = 0; i < 2 * size; ++i) tr->t[i] = -1.0;
  for (int64_t i = 0; i < n; ++i) tr->t[size + i] = v[i];
  for (int64_t i = size - 1; i > 0; --i) {
    real l = tr->t[2 * i], r = tr->t[2 * i + 1];
    tr->t[i] = l >= r ? l : r;
  }
}

static inline void tree_update(tree_t* tr, int64_t idx, real value) {
  if (!tr || tr->size == 0) return;
  int64_t i = tr->size + idx;
  tr->t[i] = value;
  i >>= 1;
  while (i >= 1) {
    real l = tr->t[2 * i], r = tr->t[2 * i + 1];
    tr->t[i] = l >= r ? l : r;
    i >>= 1;
  }
}

static inline int64_t tree_argmax(const tree_t* tr) {
  int64_t i = 1;
  while (i < tr->size) i = tr->t[2 * i] >= tr->t[2 * i + 1] ? 2 * i : 2 * i + 1;
  return i - tr->size;
}

/* E:260-276 */
static int64_t argmax_all(const real* v, int64_t n) {
  int64_t best = 0;
  for (int64_t i = 1; i < n; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

static int64_t argmax_vn_edges(const real* res, const graph_t* g, int64_t n) {
  int64_t best = g->vn_edges[g->vn_ptr[n]];
  for (int64_t k = g->vn_ptr[n] + 1; k < g->vn_ptr[n + 1]; ++k) {
    int64_t e = g->vn_edges[k];
    if (res[e] > res[best]) best = e;
  }
  return best;
}

/* ------------------------------------------------------ near-tie logging */

/* relative top-2 gap; values under GAP_FLOOR sit at the float64 noise floor of
 * the messages (1 ulp of a +-30 LLR is 3.6e-15), so the gap is taken relative
 * to max(best, GAP_FLOOR) */
#define GAP_FLOOR 1e-8
static inline void gap_note(state_t* s, double best, double second) {
  if (!s->log) return;
  if (second < 0) second = 0;
  double den = best > GAP_FLOOR ? best : GAP_FLOOR;
  double gap = (best - second) / den;
  if (gap < s->cur_gap) s->cur_gap = gap;
}

/* top-2 over a full array, for logging */
static void gap_all(state_t* s, const real* v, int64_t n) {
  if (!s->log || n < 2) return;
  double b = -1, c = -1;
  for (int64_t i = 0; i < n; ++i) {
    double x = v[i];
    if (x > b) { c = b; b = x; } else if (x > c) c = x;
  }
  gap_note(s, b, c);
}

static void gap_vn_edges(state_t* s, const real* res, const graph_t* g, int64_t n) {
  if (!s->log) return;
  double b = -1, c = -1;
  int64_t d = g->vn_ptr[n + 1] - g->vn_ptr[n];
  if (d < 2) return;
  for (int64_t k = g->vn_ptr[n]; k < g->vn_ptr[n + 1]; ++k) {
    double x = res[g->vn_edges[k]];
    if (x > b) { c = b; b = x; } else if (x > c) c = x;
  }
  gap_note(s, b, c);
}

/* test-only state dump: ci[] and pre_total[] before update `g_dump_step` */
static int64_t g_dump_step = -1;
static double *g_dump_ci = NULL, *g_dump_pt = NULL;
static int64_t g_dump_n = 0;
static double *g_dump_pre = NULL, *g_dump_c2v = NULL;
static int64_t g_dump_e = 0;
void or_set_dump_edges(double* pre, double* c2v, int64_t e) { g_dump_pre = pre; g_dump_c2v = c2v; g_dump_e = e; }
void or_set_dump(int64_t step, double* ci, double* pt, int64_t n) {
  g_dump_step = step; g_dump_ci = ci; g_dump_pt = pt; g_dump_n = n;
}
/* test-only: RNG state after each Alg.-4 selection */
static int64_t* g_rng_log = NULL;
static int64_t g_rng_cap = 0, g_rng_len = 0;
void or_set_rng_log(int64_t* buf, int64_t cap) { g_rng_log = buf; g_rng_cap = cap; g_rng_len = 0; }
int64_t or_rng_log_len(void) { return g_rng_len; }

static inline void log_step(state_t* s, int64_t e, real c2v) {
  steplog_t* L = s->log;
  if (!L) return;
  if (L->len < L->cap) {
    L->edge[L->len] = e;
    L->c2v[L->len] = (double)c2v;
    L->gap[L->len] = s->cur_gap;
  }
  L->len++;
  s->cur_gap = 1e300;
}

/* ------------------------------------------------- propagate (E:130-176) */

static void propagate(int64_t e_star, const graph_t* g, int kernel, state_t* s, int maintain_ci,
                      tree_t* res_tree, tree_t* ci_tree) {
  if (s->log && s->log->len == g_dump_step && g_dump_ci)
    for (int64_t n = 0; n < g_dump_n; ++n) { g_dump_ci[n] = (double)s->ci[n]; g_dump_pt[n] = (double)s->pre_total[n]; }
  if (s->log && s->log->len == g_dump_step && g_dump_pre)
    for (int64_t e = 0; e < g_dump_e; ++e) { g_dump_pre[e] = (double)s->pre[e]; g_dump_c2v[e] = (double)s->c2v[e]; }
  int64_t m_star = g->edge_cn[e_star];
  int64_t n_star = g->edge_vn[e_star];
  real old = s->c2v[e_star];
  s->c2v[e_star] = s->pre[e_star];
  s->res[e_star] = 0.0;
  tree_update(res_tree, e_star, 0.0);
  s->total[n_star] += s->c2v[e_star] - old;
  if (maintain_ci) {
    s->ci[n_star] = ci_of(s->total[n_star], s->pre_total[n_star]);
    tree_update(ci_tree, n_star, s->ci[n_star]);
  }
  s->counters[C_PROP] += 1;
  log_step(s, e_star, s->c2v[e_star]);
  for (int64_t k = g->vn_ptr[n_star]; k < g->vn_ptr[n_star + 1]; ++k) {
    int64_t f = g->vn_edges[k];
    int64_t i = g->edge_cn[f];
    if (i == m_star) continue;
    s->v2c[f] = clampv(s->total[n_star] - s->c2v[f]);
    s->th[f] = R_TANH((real)0.5 * s->v2c[f]);
    s->counters[C_V2C] += 1;
    for (int64_t gg = g->cn_ptr[i]; gg < g->cn_ptr[i + 1]; ++gg) {
      int64_t j = g->edge_vn[gg];
      if (j == n_star) continue;
      real old_pre = s->pre[gg];
      s->pre[gg] = cn_msg_cached(s->th, s->v2c, g, i, gg, kernel);
      s->res[gg] = R_ABS(s->pre[gg] - s->c2v[gg]);
      tree_update(res_tree, gg, s->res[gg]);
      s->counters[C_PRE] += 1;
      s->pre_total[j] += s->pre[gg] - old_pre;
      if (maintain_ci) {
        s->ci[j] = ci_of(s->total[j], s->pre_total[j]);
        tree_update(ci_tree, j, s->ci[j]);
        s->counters[C_CI] += 1;
      }
    }
  }
}

/* ---------------------------------------------- boundaries (E:179-217) */

static int syndrome_ok(const real* total, const graph_t* g) {
  uint8_t* par = (uint8_t*)calloc((size_t)g->n_checks, 1);
  for (int64_t e = 0; e < g->n_edges; ++e)
    if (total[g->edge_vn[e]] < (real)0.0) par[g->edge_cn[e]] ^= 1;
  int ok = 1;
  for (int64_t m = 0; m < g->n_checks; ++m)
    if (par[m]) { ok = 0; break; }
  free(par);
  return ok;
}

static void record_boundary(int64_t k, const graph_t* g, int64_t k_info, state_t* s) {
  int64_t errs = 0, errs_info = 0;
  for (int64_t n = 0; n < g->n_vars; ++n)
    if (s->total[n] < (real)0.0) {
      errs++;
      if (n < k_info) errs_info++;
    }
  s->biterr[k] = errs;
  s->biterr_info[k] = errs_info;
  if (s->trace) {
    int64_t N = g->n_vars;
    for (int64_t n = 0; n < N; ++n) {
      s->trace[k * 2 * N + n] = (double)s->total[n];
      s->trace[k * 2 * N + N + n] = (double)s->pre_total[n];
    }
  }
}

static void fill_remaining(int64_t k, int i_max, const graph_t* g, state_t* s) {
  for (int64_t kk = k + 1; kk <= i_max; ++kk) {
    s->biterr[kk] = s->biterr[k];
    s->biterr_info[kk] = s->biterr_info[k];
    if (s->trace) memcpy(s->trace + kk * 2 * g->n_vars, s->trace + k * 2 * g->n_vars,
                         sizeof(double) * 2 * g->n_vars);
  }
}

/* ----------------------------------------- RNG + VN selection (E:279-352) */

static inline int64_t rand_next(int64_t* st) {
  uint64_t x = (uint64_t)(*st) * 6364136223846793005ULL + 1442695040888963407ULL;
  *st = (int64_t)x;
  int64_t z = (int64_t)x;
  z ^= z >> 33;                                           /* arithmetic shift, int64 */
  z = (int64_t)((uint64_t)z * 0xFF51AFD7ED558CCDULL);      /* * -49064778989728563, wrapping */
  z ^= z >> 33;
  if (z < 0) z = -(z + 1);
  return z;
}

static inline int64_t ci_group(real c, int n_g) {
  int64_t gi = (int64_t)(c * (real)n_g);
  if (gi > n_g - 1) gi = n_g - 1;
  return gi;
}

/* near-tie note for Alg. 4: relative distance of ci*n_g to the nearest group
 * boundary, minimised over the candidate VNs (logging only) */
static void gap_groups(state_t* s, const real* ci, const int8_t* mask, int64_t n_vars, int n_g) {
  if (!s || !s->log) return;
  for (int64_t n = 0; n < n_vars; ++n) {
    if (!mask[n]) continue;
    double x = (double)ci[n] * n_g, r = floor(x + 0.5);
    if (r < 1.0 || r > n_g - 1) continue;
    double g = fabs(x - r) / r;
    if (g < s->cur_gap) s->cur_gap = g;
  }
}

static int64_t select_vns(const real* ci, const int8_t* mask, int64_t n_vars, int n_g, int n_p,
                          int64_t* rng, int64_t* out, state_t* st) {
  gap_groups(st, ci, mask, n_vars, n_g);
  int64_t* sizes = (int64_t*)calloc((size_t)n_g, sizeof(int64_t));
  for (int64_t n = 0; n < n_vars; ++n)
    if (mask[n]) sizes[ci_group(ci[n], n_g)]++;
  int64_t k_star = 0, cum = 0;
  for (int64_t k = 1; k <= n_g; ++k) {
    cum += sizes[n_g - k];
    if (cum <= n_p) k_star = k;
    else break;
  }
  int64_t count = 0, thr = n_g - k_star;
  for (int64_t n = 0; n < n_vars; ++n)
    if (mask[n] && ci_group(ci[n], n_g) >= thr) out[count++] = n;
  if (count < n_p && k_star < n_g) {
    int64_t fill = n_g - k_star - 1;
    int64_t* mem = (int64_t*)malloc(sizeof(int64_t) * (size_t)(sizes[fill] + 1));
    int64_t idx = 0;
    for (int64_t n = 0; n < n_vars; ++n)
      if (mask[n] && ci_group(ci[n], n_g) == fill) mem[idx++] = n;
    int64_t need = n_p - count;
    if (need > idx) need = idx;
    for (int64_t t = 0; t < need; ++t) {
      int64_t r = t + rand_next(rng) % (idx - t);
      int64_t tmp = mem[t];
      mem[t] = mem[r];
      mem[r] = tmp;
      out[count++] = mem[t];
    }
    free(mem);
  }
  if (g_rng_log && st && g_rng_len < g_rng_cap) g_rng_log[g_rng_len++] = *rng;
  /* sort ascending (insertion sort: count <= n_p) */
  for (int64_t a = 1; a < count; ++a) {
    int64_t v = out[a], b = a - 1;
    while (b >= 0 && out[b] > v) { out[b + 1] = out[b]; --b; }
    out[b + 1] = v;
  }
  free(sizes);
  return count;
}

/* ------------------------------------------------------------ schedules */

static void boundary_check(int64_t prop, int64_t E, const graph_t* g, const sched_t* c, state_t* s,
                           int* converged) {
  if (prop % E == 0) {
    int64_t k = prop / E;
    record_boundary(k, g, c->k_info, s);
    if (syndrome_ok(s->total, g)) {
      *converged = 1;
      fill_remaining(k, c->i_max, g, s);
    }
  }
}

/* E:355-385 */
static int64_t decode_rbp(const graph_t* g, const sched_t* c, state_t* s, int* conv) {
  int64_t E = g->n_edges, prop = 0;
  tree_t rt;
  tree_build(&rt, s->res, E);
  *conv = 0;
  while (prop < (int64_t)c->i_max * E) {
    gap_all(s, s->res, E);
    int64_t e = tree_argmax(&rt);
    s->counters[C_CMP] += E - 1;
    propagate(e, g, c->kernel, s, 0, &rt, NULL);
    prop++;
    boundary_check(prop, E, g, c, s, conv);
    if (*conv) break;
  }
  free(rt.t);
  return prop;
}

/* E:388-433 */
static int64_t decode_cirbp(const graph_t* g, const sched_t* c, state_t* s, int* conv, int64_t* kh,
                            int64_t* kt) {
  int64_t E = g->n_edges, N = g->n_vars, prop = 0;
  tree_t rt, ct;
  tree_build(&rt, s->res, E);
  tree_build(&ct, s->ci, N);
  *conv = 0;
  while (prop < (int64_t)c->i_max * E) {
    int64_t it = prop / E;
    gap_all(s, s->ci, N);
    int64_t n_star = tree_argmax(&ct);
    s->counters[C_CMP] += N - 1;
    s->counters[C_CMP] += 1;
    s->counters[C_KTRIALS] += 1;
    kt[it] += 1;
    int64_t e;
    if (s->ci[n_star] < (real)c->gamma) {
      s->counters[C_KHITS] += 1;
      kh[it] += 1;
      gap_all(s, s->res, E);
      e = tree_argmax(&rt);
      s->counters[C_CMP] += E - 1;
    } else {
      gap_vn_edges(s, s->res, g, n_star);
      e = argmax_vn_edges(s->res, g, n_star);
      s->counters[C_CMP] += (g->vn_ptr[n_star + 1] - g->vn_ptr[n_star]) - 1;
    }
    propagate(e, g, c->kernel, s, 1, &rt, &ct);
    prop++;
    boundary_check(prop, E, g, c, s, conv);
    if (*conv) break;
  }
  free(rt.t);
  free(ct.t);
  return prop;
}

/* E:436-469 */
static int64_t lmd_next_edge(const graph_t* g, const real* res, int64_t e_prev, int simplified,
                             int64_t* counters, state_t* s) {
  int64_t m_star = g->edge_cn[e_prev], n_star = g->edge_vn[e_prev];
  int deg1 = (g->vn_ptr[n_star + 1] - g->vn_ptr[n_star]) == 1;
  int64_t best = -1, ncand = 0;
  double b1 = -1, b2 = -1;
  for (int64_t k = g->vn_ptr[n_star]; k < g->vn_ptr[n_star + 1]; ++k) {
    int64_t f = g->vn_edges[k], i = g->edge_cn[f];
    if (!deg1 && i == m_star) continue;
    for (int64_t gg = g->cn_ptr[i]; gg < g->cn_ptr[i + 1]; ++gg) {
      if (g->edge_vn[gg] == n_star) continue;
      if (best < 0 || res[gg] > res[best]) best = gg;
      ncand++;
      double x = res[gg];
      if (x > b1) { b2 = b1; b1 = x; } else if (x > b2) b2 = x;
    }
  }
  if (ncand > 1) {
    counters[C_CMP] += ncand - 1;
    gap_note(s, b1, b2);
  }
  if (best < 0) return -1;
  if (!simplified) {
    int64_t np_ = g->edge_vn[best];
    gap_vn_edges(s, res, g, np_);
    best = argmax_vn_edges(res, g, np_);
    counters[C_CMP] += (g->vn_ptr[np_ + 1] - g->vn_ptr[np_]) - 1;
  }
  return best;
}

/* E:472-510 */
static int64_t decode_lmdrbp(const graph_t* g, const sched_t* c, state_t* s, int* conv,
                             int simplified) {
  int64_t E = g->n_edges, prop = 0;
  *conv = 0;
  gap_all(s, s->res, E);
  int64_t e = argmax_all(s->res, E);
  s->counters[C_CMP] += E - 1;
  while (prop < (int64_t)c->i_max * E) {
    propagate(e, g, c->kernel, s, 0, NULL, NULL);
    prop++;
    boundary_check(prop, E, g, c, s, conv);
    if (*conv) break;
    if (prop >= (int64_t)c->i_max * E) break;
    int64_t en = lmd_next_edge(g, s->res, e, simplified, s->counters, s);
    if (en < 0) {
      gap_all(s, s->res, E);
      en = argmax_all(s->res, E);
      s->counters[C_CMP] += E - 1;
    }
    e = en;
  }
  return prop;
}

/* E:513-552 ; `seen` is caller scratch of N bytes, all zero on entry and exit */
static int64_t ci_argmax_twohop(const graph_t* g, const real* ci, int64_t e_prev, int64_t* counters,
                                uint8_t* seen, state_t* s) {
  int64_t m_star = g->edge_cn[e_prev], n_star = g->edge_vn[e_prev];
  int deg1 = (g->vn_ptr[n_star + 1] - g->vn_ptr[n_star]) == 1;
  int64_t best = -1, ncand = 0;
  double b1 = -1, b2 = -1;
  if (deg1) {
    for (int64_t gg = g->cn_ptr[m_star]; gg < g->cn_ptr[m_star + 1]; ++gg) {
      int64_t j = g->edge_vn[gg];
      if (j == n_star) continue;
      if (best < 0 || ci[j] > ci[best] || (ci[j] == ci[best] && j < best)) best = j;
      ncand++;
      double x = ci[j];
      if (x > b1) { b2 = b1; b1 = x; } else if (x > b2) b2 = x;
    }
  } else {
    for (int64_t k = g->vn_ptr[n_star]; k < g->vn_ptr[n_star + 1]; ++k) {
      int64_t f = g->vn_edges[k], i = g->edge_cn[f];
      if (i == m_star) continue;
      for (int64_t gg = g->cn_ptr[i]; gg < g->cn_ptr[i + 1]; ++gg) {
        int64_t j = g->edge_vn[gg];
        if (j == n_star || seen[j]) continue;
        seen[j] = 1;
        if (best < 0 || ci[j] > ci[best] || (ci[j] == ci[best] && j < best)) best = j;
        ncand++;
        double x = ci[j];
        if (x > b1) { b2 = b1; b1 = x; } else if (x > b2) b2 = x;
      }
    }
    /* reset seen */
    for (int64_t k = g->vn_ptr[n_star]; k < g->vn_ptr[n_star + 1]; ++k) {
      int64_t f = g->vn_edges[k], i = g->edge_cn[f];
      if (i == m_star) continue;
      for (int64_t gg = g->cn_ptr[i]; gg < g->cn_ptr[i + 1]; ++gg) seen[g->edge_vn[gg]] = 0;
    }
  }
  if (ncand > 1) {
    counters[C_CMP] += ncand - 1;
    gap_note(s, b1, b2);
  }
  return best;
}

/* E:555-598 */
static int64_t decode_lmd_cirbp(const graph_t* g, const sched_t* c, state_t* s, int* conv) {
  int64_t E = g->n_edges, N = g->n_vars, prop = 0;
  uint8_t* seen = (uint8_t*)calloc((size_t)N, 1);
  *conv = 0;
  gap_all(s, s->ci, N);
  int64_t n_star = argmax_all(s->ci, N);
  s->counters[C_CMP] += N - 1;
  gap_vn_edges(s, s->res, g, n_star);
  int64_t e = argmax_vn_edges(s->res, g, n_star);
  s->counters[C_CMP] += (g->vn_ptr[n_star + 1] - g->vn_ptr[n_star]) - 1;
  while (prop < (int64_t)c->i_max * E) {
    propagate(e, g, c->kernel, s, 1, NULL, NULL);
    prop++;
    boundary_check(prop, E, g, c, s, conv);
    if (*conv) break;
    if (prop >= (int64_t)c->i_max * E) break;
    int64_t nn = ci_argmax_twohop(g, s->ci, e, s->counters, seen, s);
    if (nn < 0) {
      gap_all(s, s->ci, N);
      nn = argmax_all(s->ci, N);
      s->counters[C_CMP] += N - 1;
    }
    gap_vn_edges(s, s->res, g, nn);
    e = argmax_vn_edges(s->res, g, nn);
    s->counters[C_CMP] += (g->vn_ptr[nn + 1] - g->vn_ptr[nn]) - 1;
  }
  free(seen);
  return prop;
}

/* ME boundary loop, E:633-642 / E:681-690 */
static void me_boundaries(int64_t prop, int64_t E, const graph_t* g, const sched_t* c, state_t* s,
                          int64_t* boundary, int* conv) {
  while (*boundary <= c->i_max && prop >= *boundary * E) {
    record_boundary(*boundary, g, c->k_info, s);
    if (syndrome_ok(s->total, g)) {
      *conv = 1;
      fill_remaining(*boundary, c->i_max, g, s);
    }
    (*boundary)++;
    if (*conv) break;
  }
}

/* E:601-643 */
static int64_t decode_me_cirbp(const graph_t* g, const sched_t* c, state_t* s, int* conv) {
  int64_t E = g->n_edges, N = g->n_vars, prop = 0, boundary = 1;
  int64_t rng = c->seed;
  int8_t* mask = (int8_t*)malloc((size_t)N);
  memset(mask, 1, (size_t)N);
  int64_t* sel = (int64_t*)malloc(sizeof(int64_t) * (size_t)c->n_p);
  *conv = 0;
  while (boundary <= c->i_max && !*conv) {
    int64_t count = select_vns(s->ci, mask, N, c->n_g, c->n_p, &rng, sel, s);
    s->counters[C_MSEL] += c->n_g;
    for (int64_t idx = 0; idx < count; ++idx) {
      int64_t p = sel[idx];
      gap_vn_edges(s, s->res, g, p);
      int64_t e = argmax_vn_edges(s->res, g, p);
      s->counters[C_CMP] += (g->vn_ptr[p + 1] - g->vn_ptr[p]) - 1;
      propagate(e, g, c->kernel, s, 1, NULL, NULL);
      prop++;
    }
    me_boundaries(prop, E, g, c, s, &boundary, conv);
  }
  free(mask);
  free(sel);
  return prop;
}

/* E:646-716 */
static int64_t decode_me_lmd_cirbp(const graph_t* g, const sched_t* c, state_t* s, int* conv) {
  int64_t E = g->n_edges, N = g->n_vars, prop = 0, boundary = 1;
  int64_t rng = c->seed;
  int8_t* mask = (int8_t*)malloc((size_t)N);
  memset(mask, 1, (size_t)N);
  int64_t* sel = (int64_t*)malloc(sizeof(int64_t) * (size_t)c->n_p);
  int64_t* chosen = (int64_t*)malloc(sizeof(int64_t) * (size_t)c->n_p);
  int8_t* in_pp = (int8_t*)calloc((size_t)N, 1);
  uint8_t* seen = (uint8_t*)calloc((size_t)N, 1);
  *conv = 0;
  int64_t count = select_vns(s->ci, mask, N, c->n_g, c->n_p, &rng, sel, s);
  s->counters[C_MSEL] += c->n_g;
  while (boundary <= c->i_max && !*conv) {
    for (int64_t idx = 0; idx < count; ++idx) {
      int64_t p = sel[idx];
      gap_vn_edges(s, s->res, g, p);
      int64_t e = argmax_vn_edges(s->res, g, p);
      s->counters[C_CMP] += (g->vn_ptr[p + 1] - g->vn_ptr[p]) - 1;
      chosen[idx] = e;
      propagate(e, g, c->kernel, s, 1, NULL, NULL);
      prop++;
    }
    me_boundaries(prop, E, g, c, s, &boundary, conv);
    if (*conv || boundary > c->i_max) break;
    int64_t npc = 0;
    memset(in_pp, 0, (size_t)N);
    for (int64_t idx = 0; idx < count; ++idx) {
      int64_t pn = ci_argmax_twohop(g, s->ci, chosen[idx], s->counters, seen, s);
      if (pn >= 0 && !in_pp[pn]) {
        in_pp[pn] = 1;
        sel[npc++] = pn;
      }
    }
    if (npc < c->n_p) {
      for (int64_t n = 0; n < N; ++n) mask[n] = (int8_t)(1 - in_pp[n]);
      int64_t extra = select_vns(s->ci, mask, N, c->n_g, (int)(c->n_p - npc), &rng, sel + npc, s);
      s->counters[C_MSEL] += c->n_g;
      count = npc + extra;
    } else {
      count = npc;
    }
    for (int64_t a = 1; a < count; ++a) {
      int64_t v = sel[a], b = a - 1;
      while (b >= 0 && sel[b] > v) { sel[b + 1] = sel[b]; --b; }
      sel[b + 1] = v;
    }
  }
  free(mask); free(sel); free(chosen); free(in_pp); free(seen);
  return prop;
}

/* ME-RBP (new, see header).  Per round: the n_p largest residuals, ties to the
 * lowest edge id, propagated in ascending edge id.  C_CMP += E-1 per round. */
static int64_t decode_me_rbp(const graph_t* g, const sched_t* c, state_t* s, int* conv) {
  int64_t E = g->n_edges, prop = 0, boundary = 1;
  int64_t np_ = c->n_p < E ? c->n_p : E;
  int64_t* sel = (int64_t*)malloc(sizeof(int64_t) * (size_t)np_);
  *conv = 0;
  while (boundary <= c->i_max && !*conv) {
    /* top-np by (residual desc, id asc): insertion into a sorted list */
    int64_t cnt = 0;
    for (int64_t e = 0; e < E; ++e) {
      real v = s->res[e];
      if (cnt == np_ && !(v > s->res[sel[cnt - 1]])) continue;
      int64_t b = cnt < np_ ? cnt : np_ - 1;
      while (b > 0 && v > s->res[sel[b - 1]]) { sel[b] = sel[b - 1]; --b; }
      sel[b] = e;
      if (cnt < np_) cnt++;
    }
    if (s->log && cnt < E) {  /* near-tie at the selection boundary: n_p-th vs (n_p+1)-th */
      double lo = s->res[sel[cnt - 1]], hi = -1;
      for (int64_t e = 0; e < E; ++e) {
        int in = 0;
        for (int64_t q = 0; q < cnt; ++q) in |= sel[q] == e;
        if (!in && s->res[e] > hi) hi = s->res[e];
      }
      gap_note(s, lo, hi);
    }
    s->counters[C_CMP] += E - 1;
    for (int64_t a = 1; a < cnt; ++a) {
      int64_t v = sel[a], b = a - 1;
      while (b >= 0 && sel[b] > v) { sel[b + 1] = sel[b]; --b; }
      sel[b + 1] = v;
    }
    for (int64_t idx = 0; idx < cnt; ++idx) {
      propagate(sel[idx], g, c->kernel, s, 0, NULL, NULL);
      prop++;
    }
    me_boundaries(prop, E, g, c, s, &boundary, conv);
  }
  free(sel);
  return prop;
}

/* E:719-765 (+ E:768-782 for the trace pre-totals) */
static void flood_pre_totals(const graph_t* g, const real* chl, int kernel, state_t* s) {
  for (int64_t m = 0; m < g->n_checks; ++m)
    for (int64_t e = g->cn_ptr[m]; e < g->cn_ptr[m + 1]; ++e) s->pre[e] = cn_msg(s->v2c, g, m, e, kernel);
  for (int64_t n = 0; n < g->n_vars; ++n) {
    real acc = chl[n];
    for (int64_t k = g->vn_ptr[n]; k < g->vn_ptr[n + 1]; ++k) acc += s->pre[g->vn_edges[k]];
    s->pre_total[n] = acc;
    s->ci[n] = ci_of(s->total[n], s->pre_total[n]);
  }
}

static int64_t decode_flooding(const graph_t* g, const real* chl, const sched_t* c, state_t* s,
                               int* conv) {
  int64_t E = g->n_edges, N = g->n_vars;
  for (int64_t e = 0; e < E; ++e) {
    s->c2v[e] = 0.0;
    s->v2c[e] = clampv(chl[g->edge_vn[e]]);
  }
  for (int64_t n = 0; n < N; ++n) s->total[n] = chl[n];
  if (s->trace) flood_pre_totals(g, chl, c->kernel, s);
  record_boundary(0, g, c->k_info, s);
  *conv = 0;
  int64_t it = 0;
  for (it = 1; it <= c->i_max; ++it) {
    for (int64_t m = 0; m < g->n_checks; ++m)
      for (int64_t e = g->cn_ptr[m]; e < g->cn_ptr[m + 1]; ++e)
        s->pre[e] = cn_msg(s->v2c, g, m, e, c->kernel);
    for (int64_t e = 0; e < E; ++e) s->c2v[e] = s->pre[e];
    s->counters[C_PROP] += E;
    for (int64_t n = 0; n < N; ++n) {
      real acc = chl[n];
      for (int64_t k = g->vn_ptr[n]; k < g->vn_ptr[n + 1]; ++k) acc += s->c2v[g->vn_edges[k]];
      s->total[n] = acc;
      for (int64_t k = g->vn_ptr[n]; k < g->vn_ptr[n + 1]; ++k) {
        int64_t e = g->vn_edges[k];
        s->v2c[e] = clampv(acc - s->c2v[e]);
        s->counters[C_V2C] += 1;
      }
    }
    if (s->trace) flood_pre_totals(g, chl, c->kernel, s);
    record_boundary(it, g, c->k_info, s);
    if (syndrome_ok(s->total, g)) {
      *conv = 1;
      fill_remaining(it, c->i_max, g, s);
      break;
    }
  }
  if (it > c->i_max) it = c->i_max;   /* python's for-loop variable ends at i_max */
  return c->i_max > 0 ? it * E : 0;
}

/* Layered trace pre-totals (see header): flooding pass from v2c = clamp(total - c2v).
 * v2c / pre are scratch here (every layer recomputes them before use). */
static void layered_pre_totals(const graph_t* g, const real* chl, int kernel, state_t* s) {
  for (int64_t e = 0; e < g->n_edges; ++e) s->v2c[e] = clampv(s->total[g->edge_vn[e]] - s->c2v[e]);
  flood_pre_totals(g, chl, kernel, s);
}

/* Layered (new, see header). */
static int64_t decode_layered(const graph_t* g, const real* chl, const sched_t* c, state_t* s,
                              int* conv) {
  int64_t E = g->n_edges, N = g->n_vars;
  for (int64_t e = 0; e < E; ++e) s->c2v[e] = 0.0;
  for (int64_t n = 0; n < N; ++n) s->total[n] = chl[n];
  if (s->trace) layered_pre_totals(g, chl, c->kernel, s);
  record_boundary(0, g, c->k_info, s);
  *conv = 0;
  int64_t it = 0;
  for (it = 1; it <= c->i_max; ++it) {
    for (int64_t m = 0; m < g->n_checks; ++m) {
      int64_t a = g->cn_ptr[m], b = g->cn_ptr[m + 1];
      for (int64_t e = a; e < b; ++e) s->v2c[e] = clampv(s->total[g->edge_vn[e]] - s->c2v[e]);
      for (int64_t e = a; e < b; ++e) s->pre[e] = cn_msg(s->v2c, g, m, e, c->kernel);
      for (int64_t e = a; e < b; ++e) {
        s->total[g->edge_vn[e]] += s->pre[e] - s->c2v[e];
        s->c2v[e] = s->pre[e];
      }
      s->counters[C_PROP] += b - a;
      s->counters[C_V2C] += b - a;
    }
    if (s->trace) layered_pre_totals(g, chl, c->kernel, s);
    record_boundary(it, g, c->k_info, s);
    if (syndrome_ok(s->total, g)) {
      *conv = 1;
      fill_remaining(it, c->i_max, g, s);
      break;
    }
  }
  if (it > c->i_max) it = c->i_max;
  return c->i_max > 0 ? it * E : 0;
}

/* ------------------------------------------------------------ public API */

/* One frame.  Outputs: u_hat[N], prop, converged, counters[8],
 * biterr/biterr_info[i_max+1], kappa hits/trials[i_max] (CIRBP only, may be
 * NULL otherwise), trace[(i_max+1)*2N] or NULL, optional step log. */
int or_decode(int64_t N, int64_t M, int64_t E, const int64_t* edge_cn, const int64_t* edge_vn,
              const int64_t* cn_ptr, const int64_t* vn_ptr, const int64_t* vn_edges,
              const double* chl_in, int kind, int kernel, int i_max, int64_t k_info, double gamma,
              int n_p, int n_g, int64_t seed, int8_t* u_hat, int64_t* prop_out, uint8_t* conv_out,
              int64_t* counters, int64_t* biterr, int64_t* biterr_info, int64_t* kh, int64_t* kt,
              double* trace, int64_t log_cap, int64_t* log_edge, double* log_c2v, double* log_gap,
              int64_t* log_len) {
  graph_t g = {N, M, E, edge_cn, edge_vn, cn_ptr, vn_ptr, vn_edges};
  sched_t c = {kind, kernel, i_max, n_p, n_g, k_info, gamma, seed};
  real* buf = (real*)malloc(sizeof(real) * (size_t)(5 * E + 4 * N));
  real* chl = buf + 5 * E + 3 * N;
  for (int64_t n = 0; n < N; ++n) chl[n] = (real)chl_in[n];
  steplog_t L = {log_cap, 0, log_edge, log_c2v, log_gap};
  state_t s = {buf, buf + E, buf + 2 * E, buf + 3 * E, buf + 5 * E, buf + 5 * E + N,
               buf + 5 * E + 2 * N, buf + 4 * E, counters, biterr, biterr_info, trace,
               log_cap > 0 ? &L : NULL, 1e300};
  memset(s.pre_total, 0, sizeof(real) * (size_t)N);
  memset(s.ci, 0, sizeof(real) * (size_t)N);
  for (int k = 0; k < N_COUNTERS; ++k) counters[k] = 0;
  for (int k = 0; k <= i_max; ++k) biterr[k] = biterr_info[k] = 0;
  if (kh) for (int k = 0; k < i_max; ++k) kh[k] = kt[k] = 0;
  if (trace) memset(trace, 0, sizeof(double) * (size_t)((i_max + 1) * 2 * N));
  int conv = 0;
  int64_t prop = 0;
  if (kind == KIND_FLOODING) {
    prop = decode_flooding(&g, chl, &c, &s, &conv);
  } else if (kind == KIND_LAYERED) {
    prop = decode_layered(&g, chl, &c, &s, &conv);
  } else {
    init_state(chl, &g, kernel, &s);
    record_boundary(0, &g, k_info, &s);
    switch (kind) {
      case KIND_RBP: prop = decode_rbp(&g, &c, &s, &conv); break;
      case KIND_CIRBP: prop = decode_cirbp(&g, &c, &s, &conv, kh, kt); break;
      case KIND_LMDRBP: prop = decode_lmdrbp(&g, &c, &s, &conv, 0); break;
      case KIND_SLMDRBP: prop = decode_lmdrbp(&g, &c, &s, &conv, 1); break;
      case KIND_LMD_CIRBP: prop = decode_lmd_cirbp(&g, &c, &s, &conv); break;
      case KIND_ME_CIRBP: prop = decode_me_cirbp(&g, &c, &s, &conv); break;
      case KIND_ME_LMD_CIRBP: prop = decode_me_lmd_cirbp(&g, &c, &s, &conv); break;
      case KIND_ME_RBP: prop = decode_me_rbp(&g, &c, &s, &conv); break;
      default: free(buf); return -1;
    }
  }
  if (i_max == 0) conv = syndrome_ok(s.total, &g);   /* schedules.py:144-146 */
  for (int64_t n = 0; n < N; ++n) u_hat[n] = s.total[n] < (real)0.0 ? 1 : 0;
  *prop_out = prop;
  *conv_out = (uint8_t)conv;
  if (log_len) *log_len = L.len;
  free(buf);
  return 0;
}

/* Run or_decode over B frames on `threads` host threads (frames are
 * independent, as in the reference's process pool, sim.py:236). */
typedef struct {
  int64_t N, M, E;
  const int64_t *edge_cn, *edge_vn, *cn_ptr, *vn_ptr, *vn_edges;
  const double* chl;
  int kind, kernel, i_max, n_p, n_g;
  int64_t k_info, seed;
  double gamma;
  int8_t* u_hat;
  int64_t* prop;
  uint8_t* conv;
  int64_t *counters, *biterr, *biterr_info, *kh, *kt;
  int64_t B;
  int64_t next;
  pthread_mutex_t mu;
} batch_t;

static void* batch_worker(void* arg) {
  batch_t* b = (batch_t*)arg;
  int I = b->i_max;
  for (;;) {
    pthread_mutex_lock(&b->mu);
    int64_t f = b->next++;
    pthread_mutex_unlock(&b->mu);
    if (f >= b->B) break;
    or_decode(b->N, b->M, b->E, b->edge_cn, b->edge_vn, b->cn_ptr, b->vn_ptr, b->vn_edges,
              b->chl + f * b->N, b->kind, b->kernel, b->i_max, b->k_info, b->gamma, b->n_p, b->n_g,
              b->seed, b->u_hat + f * b->N, b->prop + f, b->conv + f, b->counters + f * N_COUNTERS,
              b->biterr + f * (I + 1), b->biterr_info + f * (I + 1),
              b->kh ? b->kh + f * (I > 0 ? I : 1) : NULL, b->kt ? b->kt + f * (I > 0 ? I : 1) : NULL,
              NULL, 0, NULL, NULL, NULL, NULL);
  }
  return NULL;
}

int or_decode_batch(int64_t B, int threads, int64_t N, int64_t M, int64_t E, const int64_t* edge_cn,
                    const int64_t* edge_vn, const int64_t* cn_ptr, const int64_t* vn_ptr,
                    const int64_t* vn_edges, const double* chl, int kind, int kernel, int i_max,
                    int64_t k_info, double gamma, int n_p, int n_g, int64_t seed, int8_t* u_hat,
                    int64_t* prop, uint8_t* conv, int64_t* counters, int64_t* biterr,
                    int64_t* biterr_info, int64_t* kh, int64_t* kt) {
  batch_t b = {N, M, E, edge_cn, edge_vn, cn_ptr, vn_ptr, vn_edges, chl, kind, kernel, i_max, n_p,
               n_g, k_info, seed, gamma, u_hat, prop, conv, counters, biterr, biterr_info, kh, kt,
               B, 0};
  pthread_mutex_init(&b.mu, NULL);
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, batch_worker, &b);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&b.mu);
  return 0;
}

/* select_vns standalone (schedules.py:60-79), for KATs */
int64_t or_select_vns(const double* ci_in, const int8_t* mask, int64_t n_vars, int n_g, int n_p,
                      int64_t seed, int64_t* out) {
  real* ci = (real*)malloc(sizeof(real) * (size_t)n_vars);
  for (int64_t n = 0; n < n_vars; ++n) ci[n] = (real)ci_in[n];
  int64_t rng = seed;
  int64_t r = select_vns(ci, mask, n_vars, n_g, n_p, &rng, out, NULL);
  free(ci);
  return r;
}

int64_t or_rand_next(int64_t* state) { return rand_next(state); }
