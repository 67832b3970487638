"""Oracle: append-only batched insertion.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Restates the reference
updater (paths relative to /root/reference/pkg/src/bucketann/updater.py):

* Eq.1/Eq.2 greedy selection          49-84
* reverse rewiring of one request     87-123
* exact in-bucket candidates          126-151
* insert orchestration                154-263
* prefix in-degree + forced healing   266-324
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .beam import beam_search, derive_seed
from .construct import build, gemm_sq, smallest_k
from .index_state import SENTINEL, OracleIndex, SearchCfg, append_rows, sqdist

LOCAL_FACTOR = 2  # updater.py:25
SEARCH_ITOPK, SEARCH_WIDTH, SEARCH_ITERS = 128, 4, 50  # updater.py:26-28


@dataclass
class InsertTally:
    """InsertReport counters (updater.py:31-46)."""

    batch_size: int = 0
    bulk_built: int = 0
    forward_accepted: int = 0
    forward_rejected: int = 0
    reverse_accepted: int = 0
    reverse_rejected: int = 0
    evictions_necessary: int = 0
    evictions_redundant: int = 0
    forced_links: int = 0
    rewired_rows: list[int] = field(default_factory=list)


def prune(X: np.ndarray, target: int, cands: list[tuple[int, float]], cap: int, alpha: float,
          fresh_from: int) -> list[int]:
    """select_neighbors (updater.py:49-84); fresh == slot >= fresh_from."""
    if not cands:
        return []
    a2 = alpha * alpha
    slots = np.array([c[0] for c in cands], dtype=np.int64)
    nearest = np.full(len(slots), np.inf)
    keep: list[int] = []
    kept: set[int] = set()
    for i, (s, d) in enumerate(cands):
        if len(keep) == cap:
            break
        if s == target or s in kept:
            continue
        de = a2 * d if s >= fresh_from else d
        if not de < nearest[i]:
            continue
        keep.append(int(s))
        kept.add(int(s))
        np.minimum(nearest, sqdist(X[s], X[slots]), out=nearest)
    return keep


def prune_set(X, target, cands, cap, alpha, fresh: set[int]) -> list[int]:
    """select_neighbors with an explicit fresh set (the reference's signature)."""
    if not cands:
        return []
    a2 = alpha * alpha
    slots = np.array([c[0] for c in cands], dtype=np.int64)
    nearest = np.full(len(slots), np.inf)
    keep: list[int] = []
    for i, (s, d) in enumerate(cands):
        if len(keep) == cap:
            break
        if s == target or s in keep:
            continue
        if not (a2 * d if s in fresh else d) < nearest[i]:
            continue
        keep.append(int(s))
        np.minimum(nearest, sqdist(X[s], X[slots]), out=nearest)
    return keep


def rewire(X: np.ndarray, A: np.ndarray, v: int, q: int, d_vq: float, alpha: float,
           k_local: int) -> tuple[bool, int]:
    """try_rewire (updater.py:87-123)."""
    row = A[v]
    if q in row:
        return False, -1
    free = np.flatnonzero(row == SENTINEL)
    if free.size:
        row[free[0]] = q
        return True, -1
    cur = row.astype(np.int64)
    if not np.all(alpha * alpha * d_vq < sqdist(X[q], X[cur])):
        return False, -1
    dv = sqdist(X[v], X[cur])
    reg = np.arange(k_local, len(row)) if len(row) > k_local else np.arange(len(row))
    p = int(reg[np.argmax(dv[reg])])
    row[p] = q
    return True, p


def local_candidates(index: OracleIndex, fresh: np.ndarray, budget: int) -> dict[int, np.ndarray]:
    """_bucket_candidates (updater.py:126-151)."""
    out: dict[int, np.ndarray] = {}
    bk = index.i2b[fresh]
    for b in np.unique(bk).tolist():
        qs = fresh[bk == b]
        mem = np.asarray(index.b2i[b], dtype=np.int64)
        D = gemm_sq(index.X[qs], index.X[mem])
        D[mem[None, :] >= qs[:, None]] = np.inf
        ids = smallest_k(D, min(budget, D.shape[1]))
        got = mem[ids]
        dd = np.take_along_axis(D, ids, axis=1)
        for r, q in enumerate(qs.tolist()):
            out[q] = got[r][np.isfinite(dd[r])]
    return out


def prefix_indegree(A: np.ndarray, prefix: int, start: int, end: int) -> np.ndarray:
    """_incoming_from_prefix (updater.py:266-271)."""
    f = A[:prefix].ravel()
    f = f[f != SENTINEL].astype(np.int64)
    f = f[(f >= start) & (f < end)]
    return np.bincount(f - start, minlength=end - start)


def heal(index: OracleIndex, start: int, end: int, nearest_pre: dict[int, int],
         touched: set[int], tally: InsertTally) -> None:
    """_heal_unreachable (updater.py:274-324)."""
    A, X, kl = index.adjacency, index.X, index.cfg.k_local
    for _ in range(4):
        miss = np.flatnonzero(prefix_indegree(A, start, start, end) == 0)
        if miss.size == 0:
            return
        for off in miss.tolist():
            q = start + off
            rq = A[q]
            t = rq[rq != SENTINEL].astype(np.int64)
            t = t[t < start]
            if t.size:
                dq = sqdist(X[q], X[t])
                v = int(t[np.lexsort((t, dq))[0]])
            elif q in nearest_pre:
                v = nearest_pre[q]
            else:
                continue
            row = A[v]
            free = np.flatnonzero(row == SENTINEL)
            if free.size:
                row[free[0]] = q
            else:
                reg = np.arange(kl, len(row)) if len(row) > kl else np.arange(len(row))
                cur = row.astype(np.int64)
                dv = sqdist(X[v], X[cur])
                stale = reg[(cur[reg] < start) | (cur[reg] >= end)]
                pool = stale if stale.size else reg
                row[int(pool[np.argmax(dv[pool])])] = q
                tally.evictions_redundant += 1
            tally.forced_links += 1
            touched.add(v)


def insert(index: OracleIndex, vectors, scalars, ids=None, search_itopk: int = SEARCH_ITOPK) -> InsertTally:
    """insert_batch (updater.py:154-263)."""
    cfg = index.cfg
    V = np.asarray(vectors, dtype=np.float32)
    S = np.asarray(scalars, dtype=np.float32)
    tally = InsertTally(batch_size=len(V))
    if index.count == 0:
        head = min(len(V), cfg.bucket_capacity)
        built, _, _ = build(V[:head], S[:head], cfg, capacity=index.capacity)
        for name in ("X", "scalars", "ids", "count", "adjacency", "boundaries", "i2b", "b2i"):
            setattr(index, name, getattr(built, name))
        tally.bulk_built = head
        if head == len(V):
            return tally
        V, S = V[head:], S[head:]
        ids = ids[head:] if ids is not None else None
    n0 = index.count
    start, end = append_rows(index, V, S, ids)
    if start == end:
        return tally
    X, A, i2b = index.X, index.adjacency, index.i2b
    fresh = np.arange(start, end, dtype=np.int64)
    local = local_candidates(index, fresh, LOCAL_FACTOR * cfg.k_max)
    requests: list[tuple[int, int, float]] = []
    touched: set[int] = set()
    nearest_pre: dict[int, int] = {}
    for q in fresh.tolist():
        cs = local.get(q, np.empty(0, np.int64))
        if n0 > 0:
            sc = SearchCfg(k=search_itopk, itopk=search_itopk, search_width=SEARCH_WIDTH,
                           max_iterations=SEARCH_ITERS, rng_seed=derive_seed(cfg.rng_seed, q))
            cs = np.union1d(cs, beam_search(index, X[q], sc, live_count=n0).slots)
        if cs.size == 0:
            continue
        d = sqdist(X[q], X[cs])
        o = np.lexsort((cs, d))
        cl = [(int(cs[i]), float(d[i])) for i in o]
        for s, _ in cl:
            if s < start:
                nearest_pre[q] = s
                break
        acc = prune(X, q, cl, cfg.k_max, cfg.alpha, start)
        tally.forward_accepted += len(acc)
        tally.forward_rejected += len(cl) - len(acc)
        if not acc:
            continue
        dmap = dict(cl)
        arr = np.array(acc, dtype=np.int64)
        same = i2b[arr] == i2b[q]
        row = np.concatenate([arr[same], arr[~same]])
        A[q, : len(row)] = row
        requests.extend((int(v), q, dmap[int(v)]) for v in row)
    requests.sort()
    for v, q, dvq in requests:
        ok, p = rewire(X, A, v, q, dvq, cfg.alpha, cfg.k_local)
        if ok:
            tally.reverse_accepted += 1
            touched.add(v)
            if p >= 0:
                if p >= cfg.k_local:
                    tally.evictions_redundant += 1
                else:
                    tally.evictions_necessary += 1
        else:
            tally.reverse_rejected += 1
    if n0 > 0:
        heal(index, start, end, nearest_pre, touched, tally)
    tally.rewired_rows = sorted(touched)
    return tally
