"""Oracle: range-constrained beam search, exact filtered brute force, recall.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Restates the reference's
search path (paths relative to /root/reference/pkg/src/bucketann):

* seed sampling          searcher.py:101-153
* queue admit/frontier   searcher.py:52-82
* Alg. 2 main loop       searcher.py:156-233
* batch seed derivation  searcher.py:85-87, 236-248
* brute force            evaluate.py:22-44
* recall / ranges        evaluate.py:47-57, 122-135

Random draws go through numpy's own Generator exactly like the reference;
oracle/rng.py restates those draws and is pinned to numpy separately.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .index_state import SENTINEL, OracleIndex, SearchCfg, bucket_interval, sqdist

_BF_BLOCK = 65_536  # evaluate.py:19


@dataclass
class Stats:
    """SearchStats counters (searcher.py:22-31) plus ``expanded`` (frontier pops)."""

    iterations: int = 0
    dist_evals: int = 0
    seed_evals: int = 0
    gathered: int = 0
    in_range_new: int = 0
    precheck_rejected: int = 0
    seed_attempts: int = 0
    expanded: int = 0


@dataclass
class Result:
    slots: np.ndarray
    sq_dists: np.ndarray
    truncated: bool
    stats: Stats = field(default_factory=Stats)


def derive_seed(base: int, ordinal: int) -> int:
    """searcher.py:85-87."""
    return int(np.random.SeedSequence([base, ordinal]).generate_state(1, np.uint64)[0])


def draw_seeds(index: OracleIndex, cfg: SearchCfg, lo: int, hi: int, n_live: int,
               gen: np.random.Generator, st: Stats) -> np.ndarray:
    """Uniform draws over buckets lo..hi, then the ordered scan fallback (searcher.py:101-153)."""
    want = cfg.want
    members = [index.b2i[b] for b in range(lo, hi + 1)]
    ends = np.cumsum([len(x) for x in members])
    total = int(ends[-1]) if len(ends) else 0
    taken: list[int] = []
    tried: set[int] = set()
    s = index.scalars

    def consider(slot: int) -> bool:
        if slot in tried or slot >= n_live:
            return False
        tried.add(slot)
        if cfg.lower <= s[slot] <= cfg.upper:
            taken.append(slot)
        return len(taken) == want

    if total > 0:
        flat = gen.integers(0, total, size=4 * want)
        st.seed_attempts += len(flat)
        for f in flat.tolist():
            b = int(np.searchsorted(ends, f, side="right"))
            if consider(members[b][f - (int(ends[b - 1]) if b else 0)]):
                break
    if len(taken) < want:
        order = [lo] + ([hi] if hi != lo else []) + list(range(lo + 1, hi))
        done = False
        for b in order:
            for slot in index.b2i[b]:
                if consider(slot):
                    done = True
                    break
            if done:
                break
    return np.array(taken, dtype=np.int64)


class Beam:
    """Bounded (dist, slot)-ordered candidate list with expansion marks (searcher.py:52-82)."""

    def __init__(self, cap: int):
        self.cap = cap
        self.slots = np.empty(0, np.int64)
        self.dists = np.empty(0, np.float64)
        self.done = np.empty(0, bool)

    def admit(self, slots, dists) -> None:
        if len(slots) == 0:
            return
        sl = np.concatenate([self.slots, slots])
        di = np.concatenate([self.dists, dists])
        dn = np.concatenate([self.done, np.zeros(len(slots), bool)])
        keep = np.lexsort((sl, di))[: self.cap]
        self.slots, self.dists, self.done = sl[keep], di[keep], dn[keep]

    def frontier(self, width: int) -> np.ndarray:
        return np.flatnonzero(~self.done)[:width]


def _empty(st: Stats) -> Result:
    return Result(np.empty(0, np.int64), np.empty(0, np.float64), False, st)


def _visit_stamps(index: OracleIndex) -> tuple[np.ndarray, int]:
    """searcher.py:90-98: an int64 stamp per row and a per-search epoch (the
    reference keeps them thread-local; the oracle is single-threaded per process)."""
    stamps = getattr(index, "_stamps", None)
    if stamps is None or len(stamps) != len(index.scalars):
        stamps = index._stamps = np.zeros(len(index.scalars), np.int64)
        index._epoch = 0
    index._epoch += 1
    return stamps, index._epoch


def beam_search(index: OracleIndex, query, cfg: SearchCfg, live_count: int | None = None) -> Result:
    """Alg. 2 (searcher.py:156-233); visited rows as epoch stamps like the reference."""
    st = Stats()
    n = index.count if live_count is None else live_count
    if n == 0 or index.boundaries is None:
        return _empty(st)
    q = np.asarray(query, dtype=np.float32)
    lo, hi = bucket_interval(index.boundaries, cfg.lower, cfg.upper)
    gen = np.random.default_rng(cfg.rng_seed)
    seeds = draw_seeds(index, cfg, lo, hi, n, gen, st)
    if len(seeds) == 0:
        return _empty(st)
    stamps, epoch = _visit_stamps(index)
    stamps[seeds] = epoch
    beam = Beam(cfg.itopk)
    beam.admit(seeds, sqdist(q, index.X[seeds]))
    st.dist_evals += len(seeds)
    st.seed_evals += len(seeds)
    s = index.scalars
    for _ in range(cfg.max_iterations):
        pos = beam.frontier(cfg.search_width)
        if pos.size == 0:
            break
        st.iterations += 1
        st.expanded += pos.size
        beam.done[pos] = True
        nb = index.adjacency[beam.slots[pos]].ravel()
        nb = nb[nb != SENTINEL].astype(np.int64)
        nb = np.unique(nb[nb < n])
        if nb.size == 0:
            continue
        st.gathered += nb.size
        new = stamps[nb] != epoch
        ok = (s[nb] >= cfg.lower) & (s[nb] <= cfg.upper)
        st.precheck_rejected += int(np.count_nonzero(new & ~ok))
        elig = nb[new & ok]
        if elig.size == 0:
            continue
        st.in_range_new += elig.size
        st.dist_evals += elig.size
        stamps[elig] = epoch
        beam.admit(elig, sqdist(q, index.X[elig]))
    k = cfg.k
    out_s, out_d = beam.slots[:k].copy(), beam.dists[:k].copy()
    return Result(out_s, out_d, 0 < len(out_s) < k, st)


def beam_search_batch(index: OracleIndex, queries, cfg: SearchCfg, live_count=None) -> list[Result]:
    """search_batch (searcher.py:236-248): per-query seed = derive(cfg.rng_seed, i)."""
    Q = np.asarray(queries, dtype=np.float32)
    return [beam_search(index, q, replace(cfg, rng_seed=derive_seed(cfg.rng_seed, i)), live_count)
            for i, q in enumerate(Q)]


def exact_filtered(index: OracleIndex, query, k: int, lower: float, upper: float,
                   live_count: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """brute_force_search (evaluate.py:22-44): stable (dist, slot) top-k of in-range rows."""
    n = index.count if live_count is None else live_count
    q = np.asarray(query, dtype=np.float32)
    s = index.scalars[:n]
    ok = np.flatnonzero((s >= lower) & (s <= upper))
    if ok.size == 0:
        return np.empty(0, np.int64), np.empty(0, np.float64)
    d = np.concatenate([sqdist(q, index.X[ok[i:i + _BF_BLOCK]]) for i in range(0, ok.size, _BF_BLOCK)])
    top = np.argsort(d, kind="stable")[:k]
    return ok[top].astype(np.int64), d[top]


def recall(result_slots, truth_slots, k: int) -> float:
    """recall_at_k (evaluate.py:47-57)."""
    t = {int(x) for x in truth_slots}
    if not t:
        return float("nan")
    return sum(1 for x in result_slots if int(x) in t) / min(k, len(t))


def window_ranges(scalars, selectivity: float, nq: int, seed: int) -> list[tuple[float, float]]:
    """generate_ranges (evaluate.py:122-135) as (lower, upper) tuples."""
    a, b = float(np.min(scalars)), float(np.max(scalars))
    w = selectivity * (b - a)
    g = np.random.default_rng([seed, 3, int(round(selectivity * 1_000_000))])
    st = a + g.random(nq) * ((b - a) - w)
    return [(float(x), float(x + w)) for x in st]
