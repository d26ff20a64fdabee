"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the tests, the bench and smoke() on BOTH sides of the
parity check (the CUDA path and the CPU oracle).  It therefore holds none of
the method's arithmetic -- no selection, softmax, capacity, layout or combine
-- only random numbers and the workload shapes (DESIGN.md §5 "input recipe").

Generator: splitmix64, used counter-style (value i of stream `seed` is
mix(seed + (i+1)*golden_gamma)), so any slice of a stream can be produced
independently and vectorised in numpy.

Workloads (BASELINE.json configs, labelled C1..C5 as in SURVEY.md §0.3):
the paper's layer is batch 32 x seq 1024 tokens, d_model 1024-2048, 8-64
experts (north_star).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
BASE_SEED = 220314685


def seed_for(config_index: int, rank: int = 0, stream: int = 0) -> int:
    """seed = 220314685 + 1000*c + r (+ 10**6 * stream for independent streams)."""
    return BASE_SEED + 1000 * config_index + rank + 1_000_000 * stream


def splitmix64(seed: int, start: int, n: int) -> np.ndarray:
    """Values start..start+n-1 of the splitmix64 stream `seed` (uint64)."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, start: int, n: int) -> np.ndarray:
    """Doubles in the open interval (0, 1): ((x >> 11) + 0.5) * 2^-53."""
    x = splitmix64(seed, start, n) >> np.uint64(11)
    return (x.astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def normal(seed: int, start: int, n: int) -> np.ndarray:
    """N(0,1) doubles by Box-Muller over consecutive uniform pairs."""
    m = (n + 1) // 2
    u = uniform(seed, 2 * start, 2 * m).reshape(m, 2)
    r = np.sqrt(-2.0 * np.log(u[:, 0]))
    th = 2.0 * np.pi * u[:, 1]
    z = np.empty((m, 2), np.float64)
    z[:, 0] = r * np.cos(th)
    z[:, 1] = r * np.sin(th)
    return z.reshape(-1)[:n]


def normal_f32(seed: int, n: int) -> np.ndarray:
    """Fast N(0,1) float32 (24-bit uniforms, float32 Box-Muller) for big x."""
    m = (n + 1) // 2
    bits = splitmix64(seed, 0, m)
    u1 = ((bits >> np.uint64(40)).astype(np.float32) + np.float32(0.5)) * np.float32(2.0 ** -24)
    u2 = (((bits >> np.uint64(8)) & np.uint64(0xFFFFFF)).astype(np.float32)) * np.float32(2.0 ** -24)
    r = np.sqrt(np.float32(-2.0) * np.log(u1))
    th = np.float32(2.0 * np.pi) * u2
    z = np.empty((m, 2), np.float32)
    np.multiply(r, np.cos(th), out=z[:, 0])
    np.multiply(r, np.sin(th), out=z[:, 1])
    return z.reshape(-1)[:n]


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Input quantisation only: float32 -> bf16 bit patterns, nearest-even
    (finite inputs).  Both sides then consume the same bf16 bits."""
    b = np.ascontiguousarray(a, np.float32).view(np.uint32)
    bias = ((b >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return ((b + bias) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return (h.astype(np.uint32) << np.uint32(16)).view(np.float32)


def _too_close(rows: np.ndarray, kind: str, k: int, gap: float) -> np.ndarray:
    """Rows whose deciding logits are within `gap` of each other (near ties):
    the top k+1 of the row (top-k), or the top 2 of each prototype slice
    (k-top-1).  Such rows are re-drawn so no near-tie logits are generated."""
    S, E = rows.shape
    if kind == "ktop1":
        sl = np.sort(rows.reshape(S, k, E // k), axis=2)
        if E // k < 2:
            return np.zeros(S, bool)
        return ((sl[:, :, -1] - sl[:, :, -2]) < gap).any(axis=1)
    m = min(k + 1, E)
    if m < 2:
        return np.zeros(S, bool)
    top = -np.sort(-rows, axis=1)[:, :m]
    return (np.diff(-top, axis=1) < gap).any(axis=1)


def logits(seed: int, S: int, E: int, k: int = 1, kind: str = "topk", gap: float = 1e-4,
           skew: float = 0.0) -> np.ndarray:
    """Gate logits [S, E] float32, i.i.d. N(0,1) (a load-balanced router in
    expectation), near-tie rows re-drawn from further down the stream.
    skew > 0 adds the expert bias -skew*ln(1+e) (a drop-stress variant)."""
    out = normal(seed, 0, S * E).astype(np.float32).reshape(S, E)
    if skew:
        out += (-skew * np.log1p(np.arange(E))).astype(np.float32)
    pos = S * E
    bad = np.nonzero(_too_close(out, kind, k, gap))[0]
    tries = 0
    while bad.size and gap > 0:
        fresh = normal(seed, pos, bad.size * E).astype(np.float32).reshape(-1, E)
        if skew:
            fresh += (-skew * np.log1p(np.arange(E))).astype(np.float32)
        pos += bad.size * E
        out[bad] = fresh
        still = _too_close(out[bad], kind, k, gap)
        bad = bad[still]
        tries += 1
        if tries > 1000:
            raise RuntimeError("could not draw tie-free logits")
    return out


def group_logits_and_logits(seed: int, S: int, E: int, k: int, n_groups: int,
                            gap: float = 1e-4):
    """Hierarchical-gate inputs: group logits [S, n_groups] (top 2 of every
    row >= gap apart) and expert logits [S, E] with the top k+1 of EVERY
    group's slice >= gap apart, so no near ties are generated whichever
    group wins (i.i.d. N(0,1); rows re-drawn like logits())."""
    gl = logits(seed, S, n_groups, 1, "topk", gap)
    n = E // n_groups
    out = normal(seed + 7, 0, S * E).astype(np.float32).reshape(S, E)
    pos = S * E

    def close(rows):
        m = min(k + 1, n)
        if m < 2:
            return np.zeros(rows.shape[0], bool)
        top = -np.sort(-rows.reshape(-1, n_groups, n), axis=2)[:, :, :m]
        return (np.diff(-top, axis=2) < gap).any(axis=(1, 2))
    bad = np.nonzero(close(out))[0]
    while bad.size:
        fresh = normal(seed + 7, pos, bad.size * E).astype(np.float32).reshape(-1, E)
        pos += bad.size * E
        out[bad] = fresh
        bad = bad[close(out[bad])]
    return gl, out


def uniforms_f32(seed: int, S: int, E: int) -> np.ndarray:
    """Uniform draws [S, E] float32 in the open interval (0, 1), for the
    Dense-to-Sparse gate's Gumbel noise: ((x >> 40) + 0.5) * 2^-24."""
    x = splitmix64(seed, 0, S * E) >> np.uint64(40)
    return ((x.astype(np.float64) + 0.5) * 2.0 ** -24).astype(np.float32).reshape(S, E)


def tokens(seed: int, S: int, d: int, dtype: str = "bf16") -> np.ndarray:
    """Token batch x_S [S, d], i.i.d. N(0,1): float32, or uint16
    bf16 bit patterns when dtype == 'bf16'."""
    x = normal_f32(seed, S * d).reshape(S, d)
    return f32_to_bf16_bits(x) if dtype == "bf16" else x


def hash_inputs(seed: int, S: int, V: int, E: int):
    """Hash-layer inputs: token ids uniform in [0, V), and
    a balanced random table = a seeded permutation of [0, V) taken mod E."""
    ids = (splitmix64(seed, 0, S) % np.uint64(V)).astype(np.int32)
    keys = splitmix64(seed + 1, 0, V)
    perm = np.argsort(keys, kind="stable").astype(np.int64)
    table = (perm % E).astype(np.int32)
    return ids, table


@dataclass
class Workload:
    """One BASELINE.json config.  S is tokens PER RANK (weak scaling)."""
    name: str
    index: int
    kind: str
    S: int
    d: int
    E: int
    k: int
    C: float
    dtype: str
    vocab: int = 0
    P: tuple = (1,)
    note: str = ""
    extra: dict = field(default_factory=dict)


WORKLOADS = {
    "C1": Workload("C1", 0, "topk", 1024, 64, 4, 1, 1.0, "f32", P=(1,),
                   note="Switch top-1, S=1024, d=64, E=4, C=1.0, fp32 (BASELINE.json configs[0])"),
    "C2": Workload("C2", 1, "topk", 32768, 1024, 8, 2, 1.0, "bf16", P=(1, 2, 4, 8),
                   note="GShard top-2, S=32x1024, d=1024, E=8, bf16 (configs[1])"),
    "C3": Workload("C3", 2, "topk", 32768, 2048, 64, 1, 1.0, "bf16", P=(1, 2, 4, 8),
                   note="Switch top-1, 32x1024 tokens, d=2048, E=64 sharded (configs[2])"),
    "C4a": Workload("C4a", 3, "ktop1", 65536, 1024, 32, 2, 1.0, "bf16", P=(8,),
                    note="k-top-1 (M6-T), 2 prototypes, S=65536, d=1024, E=32 (configs[3])"),
    "C4b": Workload("C4b", 4, "hash", 65536, 1024, 32, 1, 1.25, "bf16", vocab=32768, P=(8,),
                    note="hash gate, balanced random table V=32768, C=1.25 (configs[3])"),
    "C5": Workload("C5", 5, "topk", 32768, 1024, 64, 2, 1.0, "bf16", P=(2, 4, 8),
                   note="flat vs hierarchical (4+4) AllToAll sweep, top-2, E=64 (configs[4])"),
}


def workload_inputs(w: Workload, rank: int = 0, S: int | None = None):
    """(logits or None, token_ids or None, table or None, x) for one rank."""
    S = w.S if S is None else S
    lg = ids = table = None
    if w.kind == "hash":
        ids, table = hash_inputs(seed_for(w.index, rank, 1), S, w.vocab, w.E)
        if rank:  # one table for all ranks
            _, table = hash_inputs(seed_for(w.index, 0, 1), 1, w.vocab, w.E)
    else:
        lg = logits(seed_for(w.index, rank, 1), S, w.E, w.k, w.kind)
    x = tokens(seed_for(w.index, rank, 2), S, w.d, w.dtype)
    return lg, ids, table, x
