/*
 * heddle_place.h -- C ABI of the B200-native presorted-DP trajectory placement
 * (Heddle, arxiv 2603.28101, §5.2 "Presorted Dynamic Programming").
 *
 * Citations: "P:n" = PAPER.md line n (section / equation named alongside),
 * "S:n" = SPEC.md line n.  The meaning of every argument follows the paper's
 * problem statement (§5.1): n trajectories with lengths L sorted in
 * descending order, m rollout workers, a base per-token time T and an
 * interference factor F that depends only on the group size, per worker
 * MP degree (§6.1, sorted mapping P:703-706).
 *
 * What one solve computes, per problem (Eq. 3, stored as dp[j][i]):
 *     dp[0][0] = 0
 *     dp[j][i] = min_{k in [j-1, i-1]}  dp[j-1][k]  (+)  L[k] * G_j(i - k)
 *     G_j(s)   = T[d_j] * F[d_j][min(s, s_max) - 1]
 *     (+) = max (HEDDLE_MINMAX, Eq. 3, default) or + (HEDDLE_MINPLUS)
 *     cost  = +inf when the group exceeds the worker's cap (size > caps[j]) or
 *             its token sum Sp[i] - Sp[k] exceeds kv_caps[j]  (R6)
 *     back-pointer parent[j][i] = the LOWEST k attaining the minimum (R3)
 *     objective = dp[m][n] = the Eq. 2 makespan of the optimal
 *     contiguous partition (Lemma 1);  boundaries
 *     b_m = n,  b_{j-1} = parent[j][b_j],  0 = b_0 < b_1 < ... < b_m = n.
 * Only states on a complete m-group partition are computed: i in [j, n-m+j].
 *
 * Arithmetic per dtype (R7):
 *   HEDDLE_F32: G = fl32(T*F) (float32 T, F), cost = fl32(L*G); MINPLUS
 *               v = fmaf(L, G, dp).  MINMAX values are selections => exact
 *               w.r.t. the float32 emulation; <= 2^-23 relative vs FP64.
 *   HEDDLE_F64: G = T*F, cost = L*G, MINPLUS v = fma(L, G, dp), all double.
 *   HEDDLE_F32X (MINPLUS only): G and cost as HEDDLE_F32, v = dp + (double)cost in double.
 *   HEDDLE_U32: integer profile; G = T*F exactly (must be < 2^32); cost =
 *               L*G exactly; MINMAX objective uint32, MINPLUS objective uint64.
 *               Range guard: max L * max G < 2^32 - 65536 and L <= 65535,
 *               else the problem reports HEDDLE_E_RANGE (never a silent wrap).
 *
 * Memory / ownership: every pointer in heddle_place_problem and every output
 * pointer is a DEVICE pointer owned by the caller, borrowed for the
 * stream-ordered duration of the call; the caller keeps problem buffers alive
 * until heddle_place_backtrack() of the same solve has been enqueued and the
 * stream has passed it.  Host pointers appear only in heddle_place_config
 * (copied at init) and in heddle_place_solve_host() (copied inside the call).
 * The context owns its device workspace (dp rows, status words, cost tables),
 * sized at init from max_n / max_m / max_batch.
 *
 * Errors: every call returns a heddle_status and never aborts, throws or exits.
 * Argument errors are detected on the host before anything is enqueued, and
 * then nothing is written.  Per-problem data errors (unsorted lengths, NaN,
 * unknown degree, range) and infeasibility are detected ON THE DEVICE and
 * reported per problem in status_out[b] (heddle_status values); such a
 * problem's objective is the dtype's +inf / UINT max and its boundaries are -1.
 * solve / backtrack are asynchronous on `stream` (a cudaStream_t, NULL = the
 * legacy default stream).  A context is not thread-safe; distinct contexts are
 * independent.
 */
#ifndef HEDDLE_PLACE_H
#define HEDDLE_PLACE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HEDDLE_OK = 0,
  HEDDLE_E_INVALID = 1,        /* null pointer, n<1, m<1, B<1, sizes above the ctx limits, bad enum */
  HEDDLE_E_UNSORTED = 2,       /* lengths not non-increasing or degrees not non-increasing */
  HEDDLE_E_INFEASIBLE = 3,     /* n < m or capacities cannot cover the n trajectories        */
  HEDDLE_E_RANGE = 4,          /* NaN/inf/<=0 length or profile value, F decreasing, U32 guard */
  HEDDLE_E_UNKNOWN_DEGREE = 5, /* a worker's MP degree is not in the profile                   */
  HEDDLE_E_STATE = 6,          /* backtrack before solve, parents requested without KEEP_PARENTS      */
  HEDDLE_E_CUDA = 7,           /* a CUDA runtime call failed                                          */
  HEDDLE_E_NCCL = 8,           /* an NCCL call failed (split mode)                                    */
  HEDDLE_E_NOMEM = 9           /* device or host allocation failed                                    */
} heddle_status;

/* HEDDLE_F32X: float32 lengths and profile, costs fl32(L*fl32(T*F)) as in HEDDLE_F32, but min-plus
 * sums accumulated in float64 (dp values and the objective are double): the relative error of a
 * sum of m positive costs is then that of its terms (~2^-23), whatever m -- the FP32 sum of m =
 * 256 terms can drift towards the 1e-6 tolerance of north_star.  MINPLUS only. */
typedef enum { HEDDLE_U32 = 0, HEDDLE_F32 = 1, HEDDLE_F64 = 2, HEDDLE_F32X = 3 } heddle_dtype;
typedef enum { HEDDLE_MINMAX = 0 /* Eq. 3, default */, HEDDLE_MINPLUS = 1 } heddle_semiring;

/* config.flags */
#define HEDDLE_KEEP_PARENTS 0x1u  /* solve records every back-pointer (slower inner loop).  With
                                     the layered kernel this needs 32-bit dp values (F32, U32
                                     MINMAX); F64 / U32-MINPLUS parents need the batched kernel. */
#define HEDDLE_FORCE_BATCHED 0x2u /* always use the one-CTA-per-problem kernel (E_INVALID if n is
                                     too large for shared memory); default: chosen per call    */
#define HEDDLE_FORCE_LAYERED 0x4u /* always use the layered multi-CTA-per-problem kernel       */
#define HEDDLE_VALLEY 0x8u        /* MINMAX only (E_INVALID otherwise): solve by the valley search
                                     (SURVEY §8f N3).  With L non-increasing and F
                                     non-decreasing, max(dp[j-1][k], c_i(k)) first falls
                                     then rises in k, so each state needs O(log n) probes instead
                                     of a scan of k: O(n m log n) per problem.  Results (objective,
                                     dp rows, boundaries, parents) are bit-identical to the full
                                     scan.  One CTA per problem while n fits shared memory (about
                                     18k F32 items), else one launch per layer.  Not in split mode. */

typedef struct heddle_place_ctx heddle_place_ctx;

/* Interference profile and workspace limits.  Host memory,
 * copied at init.  Element type of T and F: float (F32), double (F64), uint32 (U32). */
typedef struct {
  int32_t device;          /* CUDA device ordinal                                          */
  int32_t dtype;           /* heddle_dtype                                                 */
  int32_t semiring;        /* heddle_semiring                                              */
  int32_t max_n;           /* largest n a solve may use (>= 1)                             */
  int32_t max_m;           /* largest m (>= 1)                                             */
  int32_t max_batch;       /* largest B (>= 1)                                             */
  int32_t num_degrees;     /* D >= 1 rows in the profile                                   */
  const int32_t* degrees;  /* [D] distinct MP degrees (e.g. {1,2,4,8}), > 0                 */
  const void* T;           /* [D] base per-token time at batch size 1, > 0          */
  const void* F;           /* [D][s_max] interference factor for batch size 1..s_max,      */
                           /*   > 0 and non-decreasing in the size; clamped beyond */
  int32_t s_max;           /* profiled range, >= 1                            */
  uint32_t flags;          /* HEDDLE_KEEP_PARENTS                                          */
} heddle_place_config;

/* A uniform-shape batch of B independent placement problems.  Device memory.
 * A stride is the element distance between consecutive problems' rows; stride
 * 0 broadcasts one row to all problems (e.g. one L swept over TP degrees). */
typedef struct {
  int32_t n;                    /* trajectories per problem, 1 <= n <= max_n                    */
  int32_t m;                    /* workers per problem, 1 <= m <= max_m  (n < m => INFEASIBLE)  */
  int32_t B;                    /* problems, 1 <= B <= max_batch                               */
  const void* lengths;          /* [B][n] dtype: predicted length L, non-increasing    */
  int64_t lengths_stride;
  const int32_t* degrees;       /* [B][m] MP degree of worker j, non-increasing    */
  int64_t degrees_stride;
  const int32_t* caps;          /* [B][m] max trajectories per worker, <0 = unbounded; or NULL  */
  int64_t caps_stride;
  const int64_t* kv_caps;       /* [B][m] max group token sum, <0 = unbounded; or NULL          */
  int64_t kv_caps_stride;
  const int32_t* weights;       /* [B][n] item weights >= 1 or NULL (= 1): an item stands for w  */
                                /*   trajectories after short-trajectory aggregation; */
                                /*   group size = sum of weights (R5); sum <= max_n (else the    */
                                /*   problem's E_RANGE).  One CTA per problem while n fits shared */
                                /*   memory, else the per-layer kernel (scan: K3 with the cost    */
                                /*   gathered per cell; HEDDLE_VALLEY: K8L).  Not in split mode   */
                                /*   (E_INVALID)                                                  */
  int64_t weights_stride;
  const int32_t* ms;            /* [B] per-problem worker count m_b in [1, m], or NULL (= m for all): a
                                 *   ragged batch, e.g. the simulated-annealing proposals of Alg. 2
                                 *   (P:748-753), whose split / merge moves change the worker count,
                                 *   evaluated in ONE launch.  Problem b uses degrees[b][0..m_b) (and
                                 *   caps / kv_caps likewise); its boundaries row holds b_0..b_{m_b}
                                 *   followed by -1 up to index m.  One-CTA-per-problem kernels only
                                 *   (n must fit shared memory; E_INVALID otherwise and in split mode).
                                 *   m_b outside [1, m] gives that problem HEDDLE_E_INVALID.         */
  const int32_t* ns;            /* [B] per-problem item count n_b in [1, n], or NULL (= n): problem b
                                 *   uses lengths[b][0..n_b) (weights likewise), e.g. the aggregated
                                 *   problems of heddle_place_aggregate, whose item counts
                                 *   differ.  Same kernel restriction and error rule as ms.          */
} heddle_place_problem;

/* Creates a context on cfg->device: copies and validates the profile (E_RANGE
 * if T/F are not positive/finite, F decreases, or a U32 product T*F >= 2^32),
 * builds the per-degree cost tables G_d[s] on the device (cost-table kernel),
 * and allocates the workspace.  *out is NULL on failure. */
heddle_status heddle_place_init(const heddle_place_config* cfg, heddle_place_ctx** out);

/* Enqueues the DP for all B problems on `stream`.
 *   objective_out : device [B]; float (F32), double (F64), uint32 (U32 MINMAX),
 *                   uint64 (U32 MINPLUS).  dp[m][n] of each problem.
 *   status_out    : device int32 [B] per-problem heddle_status, or NULL.
 * The context remembers the problem descriptor for heddle_place_backtrack(). */
heddle_status heddle_place_solve(heddle_place_ctx* ctx, const heddle_place_problem* prob,
                                 void* objective_out, int32_t* status_out, void* stream);

/* Enqueues the backtrack of the last solve.
 *   boundaries_out : device int32 [B][m+1], b_0 = 0 < ... < b_m = n (or -1s).
 *   parents_out    : device int32 [B][m][n+1] or NULL.  Row j-1 holds
 *                    parent[j][i] for i in [j, n-m+j] and -1 elsewhere.
 *                    Requires HEDDLE_KEEP_PARENTS (else E_STATE). */
heddle_status heddle_place_backtrack(heddle_place_ctx* ctx, int32_t* boundaries_out,
                                     int32_t* parents_out, void* stream);

/* Sampled states of the last solve (parity checks at sizes where the full back-pointer table
 * is not exported; sub-problem optima).  For each query q (device int32 arrays of nq entries):
 * problem qb[q], layer qj[q] in 1..m, column qi[q] (items [0, qi) in qj groups) ->
 *   dp_out[q]      = dp[qj][qi] of that problem, the dtype of objective_out (Eq. 3);
 *   parents_out[q] = parent[qj][qi], the LOWEST k in [qj-1, qi-1] attaining it (R3),
 *                    recomputed from dp row qj-1 with the solve's own arithmetic, so it equals
 *                    a stored back-pointer table bit for bit.
 * States outside the computed region (qi outside [qj, n-m+qj], R8), of failed problems, or
 * infeasible give parent -1 and dp = +inf / UINT max.  Works after every solve path (batched,
 * layered, valley, split).  The problem buffers of the solve must still be alive.  Asynchronous
 * on `stream`.  E_STATE before any solve; E_INVALID for null arrays with nq > 0 or nq < 0. */
heddle_status heddle_place_query(heddle_place_ctx* ctx, int32_t nq, const int32_t* qb, const int32_t* qj,
                                 const int32_t* qi, void* dp_out, int32_t* parents_out, void* stream);

/* End-to-end convenience with HOST buffers: copies the problem arrays (host
 * pointers, same layout as heddle_place_problem) to the device, solves,
 * backtracks, copies objective / boundaries / status back to host memory and
 * synchronises `stream`.  Pinned host memory makes the copies asynchronous.
 * When the batched kernel serves the call and B >= 512, the inputs are
 * pipelined: they are copied on an internal copy stream in chunks (~B/16
 * problems, >= 256), each chunk followed by a 4-byte ready flag, and the single
 * solve launch on `stream` starts at once, each CTA waiting for its problem's
 * chunk -- only the first chunk's copy is exposed.  The context's staging and
 * flags are reused: one solve_host at a time per context.
 * bytes_h2d / bytes_d2h (may be NULL) receive the bytes copied each way. */
heddle_status heddle_place_solve_host(heddle_place_ctx* ctx, const heddle_place_problem* host_prob,
                                      void* objective_host, int32_t* boundaries_host,
                                      int32_t* status_host, void* stream,
                                      int64_t* bytes_h2d, int64_t* bytes_d2h);

/* Number of kernels this context has launched since init (for bench evidence). */
int64_t heddle_place_launch_count(const heddle_place_ctx* ctx);

/* Algorithmic transitions W(n, m) of one problem: the (state, split) pairs the
 * DP evaluates on the computed region:
 * W = 2(n-m+1) + (m-2)(n-m+1)(n-m+2)/2 for m >= 2, W(n,1) = 1, 0 if n < m. */
int64_t heddle_place_transitions(int32_t n, int32_t m);

/* ---- multi-GPU split mode (one large instance) -------------------------
 * The columns of every DP layer are dealt to `world` ranks in zigzag order of
 * 512-column blocks (rank r owns blocks r and 2P-1-r of every group of 2P, which
 * balances the triangular work); each rank computes its blocks with the persistent
 * layered kernel, and the tile that completes a block stores the block's final dp
 * values straight into every peer's copy of the row over NVLink (CUDA-IPC peer memory,
 * opened at init) and then bumps the peer's per-block ready counter (system-scope
 * release): the exchange is fused into the DP kernel, with no NCCL call, pack or
 * unpack on the path.  A consumer tile on any rank waits only for the blocks of row
 * j-1 its split range covers.  HEDDLE_PLACE_EXCHANGE=nccl in the environment selects
 * the baseline instead: one launch per layer and one ncclAllGather of the packed row.
 * Every rank then holds every dp row, so objective and boundaries are identical on
 * all ranks (and bit-identical to a single-GPU solve).
 * heddle_place_solve / _backtrack are collective: all ranks call them with the same
 * problem.  HEDDLE_KEEP_PARENTS is not available in split mode (E_INVALID).
 *
 * heddle_place_nccl_unique_id: fills `bytes` >= 128 bytes (an ncclUniqueId) on one
 *   rank; the caller broadcasts it (e.g. torch.distributed) to every rank.
 * heddle_place_init_split: like heddle_place_init on cfg->device, plus
 *   ncclCommInitRank(world, id, rank).  nccl_unique_id == NULL with rank 0 selects
 *   the single-device EMULATION (all virtual ranks computed on this GPU, exchange
 *   by copy) used to test the ownership / packing logic without NCCL.
 * heddle_place_split_blocks: host-only; writes the column blocks rank owns out of
 *   ncb (up to cap entries) and returns how many it owns (-1 on bad arguments). */
heddle_status heddle_place_nccl_unique_id(void* id_out, int32_t bytes);
heddle_status heddle_place_init_split(const heddle_place_config* cfg, const void* nccl_unique_id, int32_t rank,
                                      int32_t world, heddle_place_ctx** out);
int32_t heddle_place_split_blocks(int32_t ncb, int32_t world, int32_t rank, int32_t* blocks_out, int32_t cap);
/* heddle_place_split_plan: host-only; per problem of an (n, m) solve, the number of (layer, block)
 *   pieces of the dp rows that `rank` publishes to each peer (*publishes_out) and the number it
 *   receives from the peers and waits for (*arrivals_out).  Returns 0, or -1 on bad arguments. */
int32_t heddle_place_split_plan(int32_t n, int32_t m, int32_t world, int32_t rank, int64_t* publishes_out,
                                int64_t* arrivals_out);

/* Objective only, min-max: the exact optimum dp[m][n] of each problem, bit-identical
 * to heddle_place_solve's objective, found without the O(n^2 m) DP: bisection over the ordered
 * values of X with an O(m log n) feasibility test (R_j = prefix ends coverable by exactly j groups
 * each costing <= X is an interval because the group cost is monotone in both ends; DESIGN.md §5
 * P6).  No partition is produced (backtrack after it returns E_STATE).  One warp per problem.
 * E_INVALID for HEDDLE_MINPLUS contexts, weighted items (the interval argument needs unit
 * weights) and split-mode contexts.  Same per-problem status_out / +inf conventions as solve. */
heddle_status heddle_place_objective(heddle_place_ctx* ctx, const heddle_place_problem* prob, void* objective_out,
                                     int32_t* status_out, void* stream);

/* ---- short-trajectory aggregation (§5.2) ----
 * heddle_place_aggregate: for each of B sorted problems (lengths [B][n] of `dtype`, row stride
 *   lengths_stride, non-increasing as the solve requires), the trajectories with length >=
 *   threshold stay single items and the shorter ones (a suffix) are cut into consecutive buckets
 *   of at most `bucket`; a bucket is ONE item: length = its first (largest) member, weight = its
 *   cardinality (group size = sum of weights, R5).  threshold <= 0: identity.
 *   Outputs (device): agg_lengths_out [B][n] (dtype) and weights_out [B][n] (rows filled up to
 *   n_b', padded after), starts_out [B][n+1] (first trajectory of each item, starts[n_b'] = n),
 *   n_out [B] = n_b'.  Feed them to heddle_place_solve as lengths / weights with ns = n_out.
 * heddle_place_expand: boundaries of the aggregated solve [B][m+1] -> trajectory boundaries
 *   (b_j -> starts[b_j], -1 kept).  Both asynchronous on `stream`, no context needed; E_INVALID on
 *   null pointers, n, B, m or bucket < 1, a negative stride, a NaN threshold or an unknown dtype. */
heddle_status heddle_place_aggregate(int32_t dtype, const void* lengths, int64_t lengths_stride, int32_t n, int32_t B,
                                    double threshold, int32_t bucket, void* agg_lengths_out, int32_t* weights_out,
                                    int32_t* starts_out, int32_t* n_out, void* stream);
heddle_status heddle_place_expand(const int32_t* agg_boundaries, int32_t m, int32_t B, const int32_t* starts, int32_t n,
                                  int32_t* boundaries_out, void* stream);

/* ---- device-resident resource manager: Sort-Initialized Simulated Annealing,
 * Alg. 2, P independent chains over sorted MP-degree allocations.  Per
 * iteration, all on `stream` with no host round trip (one CUDA graph replayed per iteration):
 *   perturb one thread per live chain: kind = floor(3 u0), falling through split ->
 *            merge -> redistribute when inapplicable (R13); candidates in descending
 *            degree order picked by floor(u * count) with u1 (and u2 for the redistribute
 *            alternative); split / merge change the worker count within [m_min, m_max] (R14);
 *            a proposal with more workers than n keeps the current state;
 *   evaluate ONE ragged heddle_place_solve (or heddle_place_objective when
 *            objective_only) over the P proposals, this context's algorithm and arithmetic;
 *   accept Metropolis: accept iff dC < 0 or u3 < exp(-dC / T); best-so-far;
 *            T <- cooling * T; a chain stops once T <= eps_frac * T0 (T0 = its start makespan).
 * The allowed degrees are the profile's.  Uniforms are inputs (R16): [P][iters][4] doubles
 * (kind, first pick, second pick, acceptance).  The start states come from the caller (sorted
 * degree rows padded to m_max, counts init_m).  One host synchronisation after the start states
 * are evaluated (the iteration count); E_INVALID for P > 1024 or > max_batch, m_max > max_m,
 * n > max_n, more than 16 profile degrees, cooling outside (0, 1), or split-mode contexts; the
 * solve's own errors are returned as they are.  A following heddle_place_backtrack is E_STATE.   */
typedef struct {
  int32_t n;                   /* trajectories; lengths: device [n] dtype, non-increasing */
  const void* lengths;
  int32_t chains;              /* P, 1..1024                                                      */
  int32_t m_min, m_max;        /* worker-count bounds; m_max is the row stride of degree rows     */
  const int32_t* init_degrees; /* device [P][m_max] start allocation per chain, non-increasing     */
  const int32_t* init_m;       /* device [P] workers of each start allocation                     */
  const double* uniforms;      /* device [P][iters][4]                                             */
  int32_t iters;               /* iteration cap (max_iters)                                        */
  double cooling;              /* alpha of T <- alpha T                                    */
  double eps_frac;             /* stop at T <= eps_frac * T0                                       */
  int32_t objective_only;      /* 1: makespans by heddle_place_objective (min-max only)            */
} heddle_place_anneal_args;

typedef struct {
  double* best_makespan;       /* device [P] best makespan per chain (as double)                   */
  int32_t* best_degrees;       /* device [P][m_max] best allocation (padded past best_m)           */
  int32_t* best_m;             /* device [P]                                                       */
  double* trace;               /* device [P][iters+1] or NULL: current makespan after each iteration */
  int32_t* accepted;           /* device [P][iters] or NULL: 1 where the iteration's move was accepted */
  int32_t* iterations;         /* host, or NULL: iterations run (the longest chain's)              */
} heddle_place_anneal_out;

heddle_status heddle_place_anneal(heddle_place_ctx* ctx, const heddle_place_anneal_args* args,
                                  heddle_place_anneal_out* out, void* stream);

/* Migration retarget (§5.3).  For each query q: problem
 * query_problem[q] with plan boundaries[b][0..m] (from heddle_place_backtrack; n = b_m), n_active[b]
 * remaining active trajectories n*, and the trajectory's 0-based rank among them by updated
 * predicted length (descending) -> worker_out[q] = the group whose range covers the rank under
 * capacities ceil(s_i * n* / n), s_i = b_{i+1} - b_i (ranks past the scaled total: worker m-1);
 * -1 for an invalid query (bad problem index, rank outside [0, n*), n* < 1).  All pointers are
 * device memory; asynchronous on `stream`; needs no context. */
heddle_status heddle_place_retarget(const int32_t* boundaries, int32_t m, int32_t B, const int32_t* n_active,
                                    const int32_t* query_problem, const int32_t* query_rank, int32_t nq,
                                    int32_t* worker_out, void* stream);

/* Debug builds only (compiled with -DHEDDLE_CHECK_BOUNDS): number of shared-memory index-range
 * violations the kernels detected so far on the current device; -1 in release builds. */
int64_t heddle_place_debug_violations(void);

void heddle_place_destroy(heddle_place_ctx* ctx);
const char* heddle_place_strerror(heddle_status s);

#ifdef __cplusplus
}
#endif
#endif /* HEDDLE_PLACE_H */
