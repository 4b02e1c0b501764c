/*
 * oracle/heddle_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct CPU implementation of Heddle's presorted
 * dynamic-programming trajectory placement (arxiv 2603.28101, §5.2).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the CUDA path under paper_2603_28101_b200/.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n.
 *
 *  - Objective, Eq. 2: min over partitions {g_1..g_m} of
 *        max_i  F(g_i) * max_{tau in g_i} L(tau) * T.
 *  - Lemma 1: on descending-sorted lengths an optimal partition
 *    into contiguous groups exists, so groups are index ranges [k, i).
 *  - State init: dp[i][1] = L(tau_1) * T * F({tau_1..tau_i}),
 *    dp[0][0] = 0.
 *  - Transition, Eq. 3:
 *        dp[i][j] = min_k max{ dp[k][j-1], L(tau_{k+1}) * T * F({tau_{k+1..i}}) }
 *    This file stores the paper's dp[i][j] as dp[j][i] (row = layer j).
 *  - F depends only on the group size; heterogeneous workers use the
 *    per-worker profile of their MP degree.
 *
 * Readings where the paper is silent (DESIGN.md "Readings" R1..R12):
 *  - R1 combine op: MINMAX (Eq. 3, the paper) or MINPLUS (north_star wording).
 *  - R2 split range: k in [j-1, i-1]; empty groups are disallowed.
 *  - R3 tie-break: strict '<' while scanning k ascending => LOWEST k wins.
 *  - R4 F beyond its profiled range is clamped at s_max.
 *  - R5 group size with aggregation weights = sum of weights.
 *  - R6 hard capacities: cost = +inf if group weight > cap_j or group token
 *    sum > kvcap_j; the token sum is Sp[i] - Sp[k] with Sp the left-to-right
 *    FP64 (exact uint64 in U32 mode) prefix sum of L.
 *  - R7 evaluation order (F64 mode): (L * T) * F, left to right as written in
 *    P:595 / P:605.  F32EMU mode emulates the float32 arithmetic the library
 *    documents: g = fl32(T*F), cost = fl32(L*g); MINPLUS v = fmaf(L, g, dp).
 *    U32 mode: exact integer arithmetic, g = T*F, cost = L*g (uint64).
 *    F32X mode (the library's "F32 costs, FP64 min-plus sums"): the
 *    cost as in F32EMU, MINPLUS v = prev + cost added in double.
 *  - R8 only the states that lie on a complete m-group partition are
 *    computed: layer j covers i in [j, n-m+j]; all others stay +inf.
 *
 * Build: gcc -O2 -fPIC -shared -ffp-contract=off -fopenmp -o liboracle.so heddle_oracle.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORA_F64 = 0, ORA_F32EMU = 1, ORA_U32 = 2, ORA_F32X = 3 };
enum { ORA_MINMAX = 0, ORA_MINPLUS = 1 };
enum { ORA_OK = 0, ORA_INVALID = 1, ORA_INFEASIBLE = 3, ORA_TOO_LARGE = 9 };

typedef struct {
  int32_t n, m;
  int32_t mode;          /* ORA_F64 / ORA_F32EMU / ORA_U32                          */
  int32_t semiring;      /* ORA_MINMAX (Eq. 3) / ORA_MINPLUS                        */
  const double* L;       /* [n] lengths, non-increasing                     */
  const int32_t* w;      /* [n] item weights (aggregation) or NULL => all 1   */
  int32_t num_degrees;   /* D                                                       */
  const double* T;       /* [D] base per-token time at batch 1              */
  const double* F;       /* [D][s_max] interference factor, F[d][s-1] for size s    */
  int32_t s_max;         /* profiled range; sizes beyond are clamped (R4)           */
  const int32_t* layer_deg; /* [m] profile row used by worker/layer j=1..m          */
  const int64_t* caps;   /* [m] max group weight, <0 => unbounded; NULL => none     */
  const double* kvcaps;  /* [m] max group token sum, <0 => unbounded; NULL => none  */
} ora_problem;

#define ORA_INF HUGE_VAL

/* ---------- prefix sums (R5, R6): plain left-to-right loops ---------- */
static int64_t* weight_prefix(const ora_problem* p) {
  int64_t* Wp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(p->n + 1));
  Wp[0] = 0;
  for (int t = 0; t < p->n; ++t) Wp[t + 1] = Wp[t] + (p->w ? p->w[t] : 1);
  return Wp;
}
static double* token_prefix(const ora_problem* p) {
  double* Sp = (double*)malloc(sizeof(double) * (size_t)(p->n + 1));
  Sp[0] = 0.0;
  if (p->mode == ORA_U32) {
    uint64_t acc = 0; /* exact integer sum, stored exactly while < 2^53 */
    for (int t = 0; t < p->n; ++t) { acc += (uint64_t)p->L[t]; Sp[t + 1] = (double)acc; }
  } else {
    for (int t = 0; t < p->n; ++t) Sp[t + 1] = Sp[t] + p->L[t];
  }
  return Sp;
}

/* Is group [k, i) admissible on layer j (1-based)?  R6. */
static int admissible(const ora_problem* p, const int64_t* Wp, const double* Sp,
                      int j, int k, int i) {
  int64_t size = Wp[i] - Wp[k];
  if (p->caps && p->caps[j - 1] >= 0 && size > p->caps[j - 1]) return 0;
  if (p->kvcaps && p->kvcaps[j - 1] >= 0 && (Sp[i] - Sp[k]) > p->kvcaps[j - 1]) return 0;
  return 1;
}

/* Profile entry index for a group of `size` on layer j: F is indexed by the
 * clamped size (R4), size counts from 1. */
static int64_t f_index(const ora_problem* p, int j, int64_t size) {
  int64_t s = size < p->s_max ? size : p->s_max;
  return (int64_t)p->layer_deg[j - 1] * p->s_max + (s - 1);
}

/* Group cost of items [k, i) on layer j: leader L[k] (the longest),
 * times T, times F(size) -- Eq. 2 group term, P:595 / P:605. */
static double group_cost_w(const ora_problem* p, const int64_t* Wp, const double* Sp,
                           int j, int k, int i) {
  if (!admissible(p, Wp, Sp, j, k, i)) return ORA_INF;
  int64_t size = Wp[i] - Wp[k];
  int d = p->layer_deg[j - 1];
  double Fv = p->F[f_index(p, j, size)];
  if (p->mode == ORA_F64) {
    return (p->L[k] * p->T[d]) * Fv;                 /* R7: (L*T)*F */
  } else if (p->mode == ORA_F32EMU || p->mode == ORA_F32X) {
    float g = (float)p->T[d] * (float)Fv;             /* fl32(T*F)   */
    float c = (float)p->L[k] * g;                     /* fl32(L*g)   */
    return (double)c;
  } else {
    uint64_t g = (uint64_t)p->T[d] * (uint64_t)Fv;    /* exact       */
    uint64_t c = (uint64_t)p->L[k] * g;
    return (double)c;                                 /* exact while < 2^53 */
  }
}

/* Combine of Eq. 3: max (paper) or + (north_star wording). */
static double combine(const ora_problem* p, const int64_t* Wp, const double* Sp,
                      double prev, int j, int k, int i) {
  double c = group_cost_w(p, Wp, Sp, j, k, i);
  if (prev == ORA_INF || c == ORA_INF) return ORA_INF;
  if (p->semiring == ORA_MINMAX) return prev > c ? prev : c;
  if (p->mode == ORA_F32EMU) {
    int d = p->layer_deg[j - 1];
    float g = (float)p->T[d] * (float)p->F[f_index(p, j, Wp[i] - Wp[k])];
    return (double)fmaf((float)p->L[k], g, (float)prev);
  }
  if (p->mode == ORA_U32) return (double)((uint64_t)prev + (uint64_t)c);
  return prev + c;
}

double ora_group_cost(const ora_problem* p, int j, int k, int i) {
  int64_t* Wp = weight_prefix(p);
  double* Sp = token_prefix(p);
  double c = group_cost_w(p, Wp, Sp, j, k, i);
  free(Wp); free(Sp);
  return c;
}

static int valid_problem(const ora_problem* p) {
  if (!p || p->n < 1 || p->m < 1 || !p->L || !p->T || !p->F || !p->layer_deg) return 0;
  if (p->s_max < 1 || p->num_degrees < 1) return 0;
  for (int j = 0; j < p->m; ++j)
    if (p->layer_deg[j] < 0 || p->layer_deg[j] >= p->num_degrees) return 0;
  return 1;
}

/*
 * The presorted DP.  dp and parent are [(m+1)][(n+1)] row-major
 * (row j = layer j), either may be NULL.  bounds is [m+1]:  b_0 = 0 < ... <
 * b_m = n, b_{j-1} = parent[j][b_j].  Returns ORA_INFEASIBLE when OPT = +inf.
 */
int ora_solve_threads(const ora_problem* p, double* dp_out, int32_t* parent_out,
                      int32_t* bounds, double* opt, int32_t nthreads);

int ora_solve(const ora_problem* p, double* dp_out, int32_t* parent_out,
              int32_t* bounds, double* opt) {
  return ora_solve_threads(p, dp_out, parent_out, bounds, opt, 1);
}

/* The same DP with the columns i of one layer shared out over `nthreads` OpenMP threads (the
 * states of a layer are independent: each reads only row j-1).  The arithmetic and the order of
 * the k loop of every state are unchanged, so the result is identical to ora_solve's.  Used to
 * write the configs[4] golden file (tests/golden/make_large_golden.py). */
int ora_solve_threads(const ora_problem* p, double* dp_out, int32_t* parent_out,
                      int32_t* bounds, double* opt, int32_t nthreads) {
  if (!valid_problem(p)) return ORA_INVALID;
  const int n = p->n, m = p->m;
  if (n < m) { *opt = ORA_INF; return ORA_INFEASIBLE; }
  size_t cells = (size_t)(m + 1) * (size_t)(n + 1);
  double* dp = (double*)malloc(sizeof(double) * cells);
  int32_t* par = (int32_t*)malloc(sizeof(int32_t) * cells);
  int64_t* Wp = weight_prefix(p);
  double* Sp = token_prefix(p);
  for (size_t c = 0; c < cells; ++c) { dp[c] = ORA_INF; par[c] = -1; }
  dp[0] = 0.0;                                               /* dp[0][0] = 0 */
  for (int j = 1; j <= m; ++j) {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1) if (nthreads > 1)
#endif
    for (int i = j; i <= n - (m - j); ++i) {                 /* R8 */
      double best = ORA_INF;
      int arg = -1;
      for (int k = j - 1; k <= i - 1; ++k) {                 /* R2 */
        double prev = dp[(size_t)(j - 1) * (n + 1) + k];
        if (prev == ORA_INF) continue;
        double v = combine(p, Wp, Sp, prev, j, k, i);
        if (v < best) { best = v; arg = k; }                 /* R3: strict '<' */
      }
      dp[(size_t)j * (n + 1) + i] = best;
      par[(size_t)j * (n + 1) + i] = arg;
    }
  }
  *opt = dp[(size_t)m * (n + 1) + n];
  int status = ORA_OK;
  if (*opt == ORA_INF) {
    status = ORA_INFEASIBLE;
    if (bounds) for (int j = 0; j <= m; ++j) bounds[j] = -1;
  } else if (bounds) {
    bounds[m] = n;
    for (int j = m; j >= 1; --j) bounds[j - 1] = par[(size_t)j * (n + 1) + bounds[j]];
  }
  if (dp_out) memcpy(dp_out, dp, sizeof(double) * cells);
  if (parent_out) memcpy(parent_out, par, sizeof(int32_t) * cells);
  free(dp); free(par); free(Wp); free(Sp);
  return status;
}

/* ---------------- brute force over contiguous partitions (pin P1) ---------------- */
typedef struct {
  const ora_problem* p;
  const int64_t* Wp;
  const double* Sp;
  int groups;          /* number of groups to place (uses layers 1..groups) */
  int end;             /* items [0, end) */
  int32_t cut[64 + 1];
  double best;
  int32_t best_cut[64 + 1];
  int64_t n_opt;
} bf_state;

static double bf_value(bf_state* s) {
  double acc = 0.0;
  for (int j = 1; j <= s->groups; ++j) acc = combine(s->p, s->Wp, s->Sp, acc, j, s->cut[j - 1], s->cut[j]);
  return acc;
}

/* Enumerate cut[1..groups-1] strictly increasing in lexicographic order. */
static void bf_rec(bf_state* s, int j) {
  if (j == s->groups) {
    s->cut[j] = s->end;
    double v = bf_value(s);
    if (v < s->best) {
      s->best = v; s->n_opt = 1;
      memcpy(s->best_cut, s->cut, sizeof(int32_t) * (size_t)(s->groups + 1));
    } else if (v == s->best && v != ORA_INF) {
      s->n_opt++;
    }
    return;
  }
  for (int c = s->cut[j - 1] + 1; c <= s->end - (s->groups - j); ++c) {
    s->cut[j] = c;
    bf_rec(s, j + 1);
  }
}

static int brute_prefix(const ora_problem* p, const int64_t* Wp, const double* Sp,
                        int groups, int end, double* opt, int32_t* cut_out, int64_t* n_opt) {
  if (groups > 64) return ORA_TOO_LARGE;
  bf_state s;
  memset(&s, 0, sizeof(s));
  s.p = p; s.Wp = Wp; s.Sp = Sp; s.groups = groups; s.end = end;
  s.best = ORA_INF; s.cut[0] = 0;
  if (end >= groups) bf_rec(&s, 1);
  *opt = s.best;
  if (cut_out) {
    if (s.best == ORA_INF) for (int j = 0; j <= groups; ++j) cut_out[j] = -1;
    else memcpy(cut_out, s.best_cut, sizeof(int32_t) * (size_t)(groups + 1));
  }
  if (n_opt) *n_opt = s.n_opt;
  return s.best == ORA_INF ? ORA_INFEASIBLE : ORA_OK;
}

/* OPT over all C(n-1, m-1) contiguous partitions; lex-first optimal cut vector;
 * number of optimal partitions.  Guard: n <= 24 (S:303-309 guards at 12 for
 * set partitions; contiguous enumeration is cheaper). */
int ora_brute_contiguous(const ora_problem* p, double* opt, int32_t* bounds_lexfirst,
                         int64_t* n_optimal) {
  if (!valid_problem(p)) return ORA_INVALID;
  if (p->n > 24) return ORA_TOO_LARGE;
  int64_t* Wp = weight_prefix(p);
  double* Sp = token_prefix(p);
  int st = brute_prefix(p, Wp, Sp, p->m, p->n, opt, bounds_lexfirst, n_optimal);
  free(Wp); free(Sp);
  return st;
}

/* Pin P2: canonical parents from brute-force prefix optima.  For every state
 * (j, i) in the computed region, OPT_bf(i, j) is found by enumeration and the
 * parent is the lowest k with combine(OPT_bf(k, j-1), cost_j(k, i)) ==
 * OPT_bf(i, j).  parent is [(m+1)][(n+1)], -1 outside the region / infeasible. */
int ora_canonical_parents_bf(const ora_problem* p, double* opt_bf, int32_t* parent) {
  if (!valid_problem(p)) return ORA_INVALID;
  if (p->n > 20) return ORA_TOO_LARGE;
  const int n = p->n, m = p->m;
  int64_t* Wp = weight_prefix(p);
  double* Sp = token_prefix(p);
  size_t cells = (size_t)(m + 1) * (size_t)(n + 1);
  for (size_t c = 0; c < cells; ++c) { opt_bf[c] = ORA_INF; parent[c] = -1; }
  opt_bf[0] = 0.0;
  for (int j = 1; j <= m; ++j)
    for (int i = j; i <= n; ++i) {
      double o;
      brute_prefix(p, Wp, Sp, j, i, &o, NULL, NULL);
      opt_bf[(size_t)j * (n + 1) + i] = o;
    }
  for (int j = 1; j <= m; ++j)
    for (int i = j; i <= n - (m - j); ++i) {
      double target = opt_bf[(size_t)j * (n + 1) + i];
      if (target == ORA_INF) continue;
      for (int k = j - 1; k <= i - 1; ++k) {
        double prev = opt_bf[(size_t)(j - 1) * (n + 1) + k];
        if (combine(p, Wp, Sp, prev, j, k, i) == target) {
          parent[(size_t)j * (n + 1) + i] = k;
          break;
        }
      }
    }
  free(Wp); free(Sp);
  return ORA_OK;
}

/* Pin P3 (Lemma 1): minimum of Eq. 2 over ALL set partitions of the
 * n items into m non-empty groups, homogeneous workers (every group costed
 * with layer 1's profile row).  MINMAX only.  Guard n <= 12. */
int ora_brute_setpartition(const ora_problem* p, double* opt) {
  if (!valid_problem(p)) return ORA_INVALID;
  if (p->n > 12 || p->m > 12) return ORA_TOO_LARGE;
  const int n = p->n, m = p->m;
  int label[12];
  double best = ORA_INF;
  int64_t total = 1;
  for (int t = 0; t < n; ++t) total *= m;
  int d = p->layer_deg[0];
  for (int64_t code = 0; code < total; ++code) {
    int64_t c = code;
    for (int t = 0; t < n; ++t) { label[t] = (int)(c % m); c /= m; }
    double worst = 0.0;
    int ok = 1;
    for (int g = 0; g < m && ok; ++g) {
      int64_t size = 0;
      double lead = 0.0, tokens = 0.0;
      for (int t = 0; t < n; ++t)
        if (label[t] == g) {
          size += p->w ? p->w[t] : 1;
          tokens += p->L[t];
          if (p->L[t] > lead) lead = p->L[t];
        }
      if (size == 0) { ok = 0; break; }                  /* non-empty groups */
      if (p->caps && p->caps[0] >= 0 && size > p->caps[0]) { worst = ORA_INF; continue; }
      if (p->kvcaps && p->kvcaps[0] >= 0 && tokens > p->kvcaps[0]) { worst = ORA_INF; continue; }
      int64_t s = size < p->s_max ? size : p->s_max;
      double Fv = p->F[(int64_t)d * p->s_max + s - 1];
      double cost = (lead * p->T[d]) * Fv;              /* Eq. 2 group term */
      if (cost > worst) worst = cost;
    }
    if (ok && worst < best) best = worst;
  }
  *opt = best;
  return best == ORA_INF ? ORA_INFEASIBLE : ORA_OK;
}

/* ------------- Pin P6: parametric search (MINMAX only) -------------
 * feasible(X): R_j = set of prefix ends coverable by exactly j non-empty
 * contiguous groups, group g on layer g, each costing <= X.  R_0 = {0}.
 * R_j is an interval [lo, hi]; for an end e > lo_{j-1} the cheapest start is
 * a = min(hi_{j-1}, e-1) because the cost of [a, e) is non-increasing in a
 * (leader L[a] non-increasing, size / tokens decreasing, F non-decreasing). */
int ora_feasible(const ora_problem* p, double X) {
  const int n = p->n, m = p->m;
  int64_t* Wp = weight_prefix(p);
  double* Sp = token_prefix(p);
  int lo = 0, hi = 0, ok = 1, interval = 1;
  for (int j = 1; j <= m && ok; ++j) {
    int nlo = -1, nhi = -1, gap = 0;
    for (int e = lo + 1; e <= n; ++e) {
      int a = hi < e - 1 ? hi : e - 1;
      double c = group_cost_w(p, Wp, Sp, j, a, e);
      if (c != ORA_INF && c <= X) {                /* inadmissible groups never fit */
        if (nlo < 0) nlo = e;
        if (gap) interval = 0;                     /* true after a false after a true */
        nhi = e;
      } else if (nlo >= 0) {
        gap = 1;
      }
    }
    if (nlo < 0) ok = 0;
    lo = nlo; hi = nhi;
  }
  free(Wp); free(Sp);
  /* With unit weights the single-item cost c(e-1, e) is non-increasing in e, which makes every
   * R_j an interval; item weights (aggregation) can break that, and then the test is undecided. */
  if (!interval) return -1;
  return ok && lo <= n && n <= hi;
}

/* Smallest X with feasible(X), by bisection over the ordered bit patterns of
 * non-negative doubles.  Equals the DP's OPT exactly (same cost values). */
int ora_parametric_opt(const ora_problem* p, double* opt) {
  if (!valid_problem(p)) return ORA_INVALID;
  if (p->semiring != ORA_MINMAX) return ORA_INVALID;
  if (p->n < p->m) { *opt = ORA_INF; return ORA_INFEASIBLE; }
  { const int f = ora_feasible(p, ORA_INF);
    if (f < 0) return ORA_INVALID;
    if (!f) { *opt = ORA_INF; return ORA_INFEASIBLE; } }
  uint64_t lo = 0, hi;
  double inf = ORA_INF;
  memcpy(&hi, &inf, sizeof(hi));
  /* invariant: feasible(bits(hi)) true; find smallest such pattern */
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    double x;
    memcpy(&x, &mid, sizeof(x));
    const int f = ora_feasible(p, x);
    if (f < 0) return ORA_INVALID;                 /* non-interval R_j: not decidable this way */
    if (f) hi = mid; else lo = mid + 1;
  }
  memcpy(opt, &hi, sizeof(*opt));
  return ORA_OK;
}

/* ---------------- batched entry (cpu_baseline / --impl reference) ----------------
 * B independent problems sharing n, m and the profile; lengths [B][n],
 * layer_deg [B][m].  Plain loop over ora_solve, OpenMP over problems only.
 * Returns the number of threads used. */
int ora_solve_batch(const ora_problem* proto, int32_t B, const double* lengths,
                    const int32_t* layer_deg, double* opt, int32_t* bounds, int32_t nthreads) {
  int used = 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
  {
#pragma omp single
    used = omp_get_num_threads();
#pragma omp for schedule(dynamic, 1)
    for (int b = 0; b < B; ++b) {
      ora_problem q = *proto;
      q.L = lengths + (size_t)b * (size_t)proto->n;
      q.layer_deg = layer_deg + (size_t)b * (size_t)proto->m;
      ora_solve(&q, NULL, NULL, bounds + (size_t)b * (size_t)(proto->m + 1), opt + b);
    }
  }
#else
  (void)nthreads;
  for (int b = 0; b < B; ++b) {
    ora_problem q = *proto;
    q.L = lengths + (size_t)b * (size_t)proto->n;
    q.layer_deg = layer_deg + (size_t)b * (size_t)proto->m;
    ora_solve(&q, NULL, NULL, bounds + (size_t)b * (size_t)(proto->m + 1), opt + b);
  }
#endif
  return used;
}
