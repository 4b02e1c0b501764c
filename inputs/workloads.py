"""Seeded synthetic inputs for the presorted-DP placement path.

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NONE of the method's arithmetic: it only draws trajectory lengths,
sorts them (the caller-side presort of P:581-583), and writes down profile
tables and degree vectors.  Group costs, prefix sums and the DP itself live
in oracle/ (CPU) and paper_2603_28101_b200/csrc/ (CUDA), independently.

Workload shapes (the paper gives shapes, not parameters):
  * coding / CodeForces-like (Pareto): per prompt base b_p ~ Pareto(1.2, x_m=600)
    tokens; per sample L = clamp(round(b_p * exp(0.5 z)), 64, 40960).  Long
    tail (Fig. 2; max > 4x median); 40K token cap;
    intra-group divergence 0.5.
  * search / HotpotQA-like (log-normal): mu_p ~ N(ln 1500, 0.5);
    L = clamp(round(exp(mu_p + 0.6 z)), 32, 40960).
  * FP32 configs use noisy *predicted* lengths L_hat = L * exp(0.5 z) (the
    prompt-only predictor noise sigma_0 = 0.5 of S:173 / S:212).
Profile (SPEC calibration S:93): T_d = 0.05 * d^-0.8 s/token, F(s) = 1 + 0.08 (s-1),
profiled for s = 1..S_MAX = 1024 and clamped beyond.  The integer
(U32) profile is T_int[d] = round(32 * d^-0.8), F_int[s] = 25 + 2 (s-1): an
integer-scaled copy with the same shape; T_int * F_int * 40960 < 2^32 - 65536.
"""
from __future__ import annotations

import dataclasses

import numpy as np

SEED_BASE = 0x48454444  # "HEDD"
DEGREES = (1, 2, 4, 8)  # MP (TP) degrees the resource manager sweeps
S_MAX = 1024
MAX_TOKENS = 40960


def rng_for(config: int, problem: int = 0) -> np.random.Generator:
    return np.random.default_rng(SEED_BASE + 1000 * config + problem)


# ----------------------------------------------------------------------------- lengths
def coding_lengths(rng: np.random.Generator, n_prompts: int, samples: int) -> np.ndarray:
    base = 600.0 * (1.0 + rng.pareto(1.2, size=n_prompts))
    z = rng.standard_normal((n_prompts, samples))
    L = np.rint(base[:, None] * np.exp(0.5 * z))
    return np.clip(L, 64, MAX_TOKENS).reshape(-1)


def search_lengths(rng: np.random.Generator, n_prompts: int, samples: int) -> np.ndarray:
    mu = rng.normal(np.log(1500.0), 0.5, size=n_prompts)
    z = rng.standard_normal((n_prompts, samples))
    L = np.rint(np.exp(mu[:, None] + 0.6 * z))
    return np.clip(L, 32, MAX_TOKENS).reshape(-1)


def predicted(rng: np.random.Generator, L: np.ndarray) -> np.ndarray:
    """Noisy prompt-only predictions, float32."""
    return (L * np.exp(0.5 * rng.standard_normal(L.shape))).astype(np.float32)


def presort(L: np.ndarray) -> np.ndarray:
    """Descending order, ties by trajectory id ascending."""
    ids = np.arange(L.shape[-1])
    order = np.lexsort((ids, -L.astype(np.float64)))
    return L[order]


def presort_rows(L: np.ndarray) -> np.ndarray:
    """Row-wise presort of a [B, n] array (stable => ties keep id order)."""
    return -np.sort(-L, axis=-1, kind="stable")


# ----------------------------------------------------------------------------- profiles
@dataclasses.dataclass
class Profile:
    degrees: tuple          # MP degree of each profile row
    T: np.ndarray           # [D] per-token time at batch 1
    F: np.ndarray           # [D, s_max] interference factor for size 1..s_max
    s_max: int
    dtype: str              # "f32" | "f64" | "u32"

    def row_of(self, degree_vec) -> np.ndarray:
        lut = {d: r for r, d in enumerate(self.degrees)}
        return np.array([lut[int(d)] for d in np.asarray(degree_vec).reshape(-1)],
                        dtype=np.int32).reshape(np.shape(degree_vec))


def float_profile(degrees=DEGREES, s_max=S_MAX, dtype="f32", slope=0.08) -> Profile:
    d = np.asarray(degrees, dtype=np.float64)
    T = 0.05 * d ** -0.8
    s = np.arange(1, s_max + 1, dtype=np.float64)
    F = np.broadcast_to(1.0 + slope * (s - 1.0), (len(degrees), s_max)).copy()
    if dtype == "f32":  # the F32 path consumes float32 tables; keep values representable
        T = T.astype(np.float32).astype(np.float64)
        F = F.astype(np.float32).astype(np.float64)
    return Profile(tuple(degrees), T, F, s_max, dtype)


def int_profile(degrees=DEGREES, s_max=S_MAX) -> Profile:
    d = np.asarray(degrees, dtype=np.float64)
    T = np.rint(32.0 * d ** -0.8)
    s = np.arange(1, s_max + 1, dtype=np.float64)
    F = np.broadcast_to(25.0 + 2.0 * (s - 1.0), (len(degrees), s_max)).copy()
    return Profile(tuple(degrees), T, F, s_max, "u32")


# ----------------------------------------------------------------------------- degrees
def sorted_degree_vectors(rng: np.random.Generator, B: int, m: int, degrees=DEGREES) -> np.ndarray:
    """Random non-increasing per-worker MP degrees (sort-initialised mapping)."""
    v = rng.choice(np.asarray(degrees, dtype=np.int32), size=(B, m))
    return -np.sort(-v, axis=1)


# ----------------------------------------------------------------------------- configs
@dataclasses.dataclass
class Batch:
    name: str
    n: int
    m: int
    lengths: np.ndarray         # [B, n] (float32 / uint32 / float64), rows non-increasing
    degrees: np.ndarray         # [B, m] int32 MP degree per worker, non-increasing
    profile: Profile
    caps: np.ndarray | None = None      # [B, m] int32, -1 = unbounded
    kv_caps: np.ndarray | None = None   # [B, m] int64, -1 = unbounded
    weights: np.ndarray | None = None   # [B, n] int32

    @property
    def B(self) -> int:
        return self.lengths.shape[0]


def _family(rng, fam, n):
    samples = 8
    prompts = (n + samples - 1) // samples
    L = coding_lengths(rng, prompts, samples) if fam == "coding" else search_lengths(rng, prompts, samples)
    return L[:n]


def config_tiny(problem: int = 0) -> Batch:
    """configs[0]: N=16 into K=4, integer costs (brute-force checkable)."""
    rng = rng_for(0, problem)
    L = presort(_family(rng, "coding", 16)).astype(np.uint32)
    prof = int_profile()
    deg = sorted_degree_vectors(rng, 1, 4)
    return Batch("tiny", 16, 4, L[None, :], deg, prof)


def config_rollout(problem: int = 0, dtype="f32") -> Batch:
    """configs[1]: 64 prompts x 8 samples (Pareto) into K=32 instances, FP32 costs."""
    rng = rng_for(1, problem)
    L = presort(predicted(rng, coding_lengths(rng, 64, 8)))
    deg = np.ones((1, 32), dtype=np.int32)
    return Batch("rollout", 512, 32, L[None, :].astype(np.float32), deg, float_profile(dtype=dtype))


def config_tp_sweep(problem: int = 0, n=4096, m=64) -> Batch:
    """configs[2]: N=4096 into K=64, swept over TP degrees {1,2,4,8} (one problem each,
    shared lengths) -- the resource manager's configuration search."""
    rng = rng_for(2, problem)
    L = presort(predicted(rng, coding_lengths(rng, n // 8, 8)))
    lengths = np.broadcast_to(L, (4, n)).astype(np.float32)
    deg = np.stack([np.full(m, d, dtype=np.int32) for d in DEGREES])
    return Batch("tp_sweep", n, m, np.ascontiguousarray(lengths), deg, float_profile())


def config_batched(B: int = 16384, n: int = 1024, m: int = 32, seed_problem: int = 0, dtype: str = "f32") -> Batch:
    """configs[3]: B independent N=1024 K=32 problems; coding / search families
    alternate; random sorted degree vectors over {1,2,4,8} (SA candidates).
    dtype "f32" (the bench): noisy predicted lengths; "f64": the same predictions unrounded;
    "u32": the true integer token lengths with the integer profile (bit-exact mode)."""
    rng = rng_for(3, seed_problem)
    prompts = n // 8
    base_c = 600.0 * (1.0 + rng.pareto(1.2, size=(B, prompts)))
    mu_s = rng.normal(np.log(1500.0), 0.5, size=(B, prompts))
    z = rng.standard_normal((B, prompts, 8))
    coding = np.clip(np.rint(base_c[:, :, None] * np.exp(0.5 * z)), 64, MAX_TOKENS)
    search = np.clip(np.rint(np.exp(mu_s[:, :, None] + 0.6 * z)), 32, MAX_TOKENS)
    fam = (np.arange(B) % 2 == 0)[:, None, None]
    L = np.where(fam, coding, search).reshape(B, n)
    Lhat = L * np.exp(0.5 * rng.standard_normal((B, n)))
    deg = sorted_degree_vectors(rng, B, m)
    if dtype == "u32":
        return Batch("batched", n, m, presort_rows(L).astype(np.uint32), deg, int_profile())
    if dtype == "f64":
        return Batch("batched", n, m, presort_rows(Lhat), deg, float_profile(dtype="f64"))
    return Batch("batched", n, m, presort_rows(Lhat.astype(np.float32)), deg, float_profile())


def config_large(problem: int = 0, n: int = 65536, m: int = 256, dtype: str = "f32") -> Batch:
    """configs[4]: single N=65536 K=256 instance (coding-like), degree 1.  dtype "u32": the true
    integer token lengths with the integer profile; "f64": the same predictions as doubles."""
    rng = rng_for(4, problem)
    true = coding_lengths(rng, n // 8, 8)
    L = presort(predicted(rng, true))
    deg = np.ones((1, m), dtype=np.int32)
    if dtype == "u32":
        return Batch("large", n, m, presort(true)[None, :].astype(np.uint32), deg, int_profile())
    if dtype == "f64":
        return Batch("large", n, m, L[None, :].astype(np.float64), deg, float_profile(dtype="f64"))
    return Batch("large", n, m, L[None, :].astype(np.float32), deg, float_profile())


def tiny_random(seed: int, n_max=16, m_max=4, allow_caps=True, allow_weights=False,
                allow_kv=False, dtype="u32") -> Batch:
    """Heavy-tie tiny instances for brute-force pins: lengths from a small set,
    short profiled ranges (clamp plateaus), random caps."""
    rng = np.random.default_rng(SEED_BASE + 777 + seed)
    n = int(rng.integers(1, n_max + 1))
    m = int(rng.integers(1, min(n, m_max) + 1))
    L = presort(rng.choice(np.array([1, 2, 3, 5, 8, 13, 40]), size=n).astype(np.float64))
    s_max = int(rng.integers(1, 6))
    degrees = DEGREES
    if dtype == "u32":
        T = rng.integers(1, 5, size=len(degrees)).astype(np.float64)
        steps = rng.integers(0, 3, size=(len(degrees), s_max))
        F = (1 + np.cumsum(steps, axis=1) - steps[:, :1]).astype(np.float64)
    else:
        T = rng.uniform(0.5, 2.0, size=len(degrees)).astype(np.float32).astype(np.float64)
        steps = rng.choice([0.0, 0.25, 0.5], size=(len(degrees), s_max))
        F = (1.0 + np.cumsum(steps, axis=1) - steps[:, :1]).astype(np.float32).astype(np.float64)
    prof = Profile(degrees, T, F, s_max, dtype)
    deg = sorted_degree_vectors(rng, 1, m)
    caps = None
    if allow_caps and rng.random() < 0.5:
        caps = rng.integers(-1, n + 1, size=(1, m)).astype(np.int32)
        caps[caps == 0] = -1
    w = None
    if allow_weights and rng.random() < 0.5:
        w = rng.integers(1, 4, size=(1, n)).astype(np.int32)
    kv = None
    if allow_kv and rng.random() < 0.5:
        kv = rng.integers(-1, int(L.sum()) + 1, size=(1, m)).astype(np.int64)
    ldt = np.uint32 if dtype == "u32" else (np.float32 if dtype == "f32" else np.float64)
    return Batch(f"tiny_random_{seed}", n, m, L[None, :].astype(ldt), deg, prof,
                 caps=caps, kv_caps=kv, weights=w)


# ----------------------------------------------------------------------------- SA randomness
def sa_uniforms(seed: int, chains: int, iters: int, init_moves: int = 8):
    """Pre-drawn uniforms for the simulated-annealing resource manager (Alg. 2): per chain
    1 + 3*init_moves for the initial state and 4 per iteration (move kind, first pick, second
    pick, acceptance).  Random numbers the method draws are inputs (R16)."""
    rng = np.random.default_rng(SEED_BASE + 5000 + seed)
    return rng.random((chains, 1 + 3 * init_moves)), rng.random((chains, iters, 4))
