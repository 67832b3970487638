"""Bucket-range sharded index over ranks (one process per GPU).

The reference is a single-process index ("Distributed communication
backend: none"); this layer is the B200 design for indexes that are split
across GPUs. Each rank owns one contiguous scalar range -- hence a contiguous
run of buckets -- and builds a self-contained GRAB index over its rows with the
unchanged single-GPU pipeline. A query batch is served by:

1. routing: query i goes to every shard whose [min, max] scalar span meets the
   query's f32-rounded range (the same NEP-50 rounding the kernels apply,
   searcher.py:136,215), so a shard that holds no in-range row never runs it;
2. the local filtered beam search (or exact brute force) over the routed
   queries, with the per-query RNG seed of the GLOBAL ordinal
   (derive_query_seed(seed_base, i), searcher.py:85-87);
3. ``grab_shard_pack``: local slots -> global ids, written into the block of the
   rank that owns the query (owner = i // B, B = ceil(nq / world));
4. one fixed-size all-to-all of those blocks (NCCL over NVLink on GPUs, gloo in
   the CPU tests);
5. ``grab_merge_topk``: each owner merges world x k candidates per query by
   (distance, global id), the reference's tie rule.

No query is replicated beyond the routing and no shard scans rows outside its
range; cross-shard edges do not exist (each shard is an independent graph), so
recall is measured against the global exact oracle (the same pipeline with the
brute-force kernel in step 2).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .api import brute_force_arrays, build_index, search_arrays
from .params import BuildParams, SearchParams


def plan_shards(scalars: np.ndarray, world: int) -> np.ndarray:
    """Equal-count scalar cuts f32[world+1]: shard r owns cuts[r] <= s < cuts[r+1]
    (the last shard also owns s == cuts[world]). Quantile rule of
    partition_buckets (layout.py:125-140): cut i = sorted[round(i * n / world)]."""
    s = np.sort(np.asarray(scalars, dtype=np.float32))
    n = len(s)
    if world < 1 or n < world:
        raise ValueError("need 1 <= world <= number of rows")
    idx = np.round(np.arange(world + 1) * n / world).astype(np.int64)
    idx[-1] = n - 1
    cuts = s[np.minimum(idx, n - 1)].astype(np.float32)
    cuts[0] = s[0]
    return cuts


def shard_of(scalars: np.ndarray, cuts: np.ndarray) -> np.ndarray:
    """Owning shard of each row: searchsorted over the interior cuts, 'right'."""
    return np.searchsorted(cuts[1:-1], np.asarray(scalars, dtype=np.float32), side="right").astype(np.int64)


def route(lower, upper, spans: np.ndarray) -> np.ndarray:
    """bool [world, nq]: shard r runs query i iff its scalar span meets the
    query range after the kernels' f32 rounding of the bounds."""
    lo = np.asarray(lower, dtype=np.float64).astype(np.float32)
    hi = np.asarray(upper, dtype=np.float64).astype(np.float32)
    smin = spans[:, 0:1].astype(np.float32)
    smax = spans[:, 1:2].astype(np.float32)
    return (lo[None, :] <= smax) & (hi[None, :] >= smin) & (smin <= smax)


def owner_block(nq: int, world: int) -> int:
    return max(1, math.ceil(nq / world))


def derive_seeds(seed_base: int, ordinals: np.ndarray) -> np.ndarray:
    o = np.ascontiguousarray(ordinals, dtype=np.uint32)
    out = np.empty(len(o), dtype=np.uint64)
    if len(o):
        L.check(L.lib.grab_derive_seeds(int(seed_base), L.ptr(o), len(o), L.ptr(out)))
    return out


@dataclass
class ShardResult:
    """Merged results of the queries this rank owns: [first, first + n)."""

    first: int
    slots: "object"  # int64 [n, k] global ids, -1 padded (torch CUDA tensor)
    dists: "object"  # float64 [n, k]
    counts: "object"  # uint32 [n] (as int32 tensor)
    routed: int  # queries this rank searched


class ShardedIndex:
    """One rank's shard plus the group-wide routing table."""

    def __init__(self, local, gid, spans: np.ndarray, rank: int, world: int, group=None, device: int = 0):
        import torch
        self.local = local
        self.rank, self.world, self.group, self.device = rank, world, group, device
        self.spans = np.asarray(spans, dtype=np.float32)
        self.gid = torch.as_tensor(np.ascontiguousarray(gid, dtype=np.int64), device=self._dev())

    def _dev(self):
        import torch
        return torch.device("cuda", self.device)

    # ------------------------------------------------------------------ build
    @classmethod
    def build(cls, X_local, S_local, gid_local, params: BuildParams, *, rank: int, world: int, group=None,
              device: int = 0, **build_kw):
        """Build this rank's shard from its own rows (already restricted to its
        scalar range) and exchange the shard spans."""
        import torch
        import torch.distributed as dist
        local, report = build_index(X_local, S_local, params, device=device, **build_kw)
        S = np.asarray(S_local.cpu().numpy() if hasattr(S_local, "cpu") else S_local, dtype=np.float32)
        mine = np.array([[S.min(), S.max()]] if len(S) else [[np.inf, -np.inf]], dtype=np.float64)
        if world > 1:
            t = torch.as_tensor(mine, device=_coll_device(group, device))
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t, group=group)
            spans = torch.cat(parts).cpu().numpy()
        else:
            spans = mine
        return cls(local, gid_local, spans, rank, world, group, device), report

    # ------------------------------------------------------------------ query
    def search(self, queries, lower, upper, params: SearchParams, *, seed_base: int | None = None,
               exact: bool = False) -> ShardResult:
        """Route, search (or brute-force when ``exact``), pack, exchange, merge.
        ``queries``/``lower``/``upper`` are the FULL batch (identical on every
        rank); the result covers the queries this rank owns."""
        import torch
        dev = self._dev()
        lower = np.asarray(lower, dtype=np.float64)
        upper = np.asarray(upper, dtype=np.float64)
        nq = len(lower)
        k = params.k
        B = owner_block(nq, self.world)
        mask = route(lower, upper, self.spans)[self.rank]
        mine = np.nonzero(mask)[0].astype(np.uint32)
        Qd = queries if hasattr(queries, "is_cuda") else torch.from_numpy(np.ascontiguousarray(queries)).to(dev)
        idx_d = torch.from_numpy(mine.astype(np.int64)).to(dev)
        Qm = Qd.index_select(0, idx_d).contiguous()
        lo_m = torch.from_numpy(lower[mine]).to(dev)
        hi_m = torch.from_numpy(upper[mine]).to(dev)
        if len(mine) == 0:
            slots = torch.empty((0, k), dtype=torch.int64, device=dev)
            dists = torch.empty((0, k), dtype=torch.float64, device=dev)
        elif exact:  # the oracle pipeline (ground truth), host-staged
            s_h, d_h, _ = brute_force_arrays(self.local, Qm.cpu().numpy(), lower[mine], upper[mine], k)
            slots, dists = torch.from_numpy(s_h).to(dev), torch.from_numpy(d_h).to(dev)
        else:
            base = params.rng_seed if seed_base is None else seed_base
            r = search_arrays(self.local, Qm, lo_m, hi_m, params, seeds=derive_seeds(base, mine), stats=False)
            slots, dists = r.slots, r.dists
        send_d = torch.empty((self.world, B, k), dtype=torch.float64, device=dev)
        send_i = torch.empty((self.world, B, k), dtype=torch.int64, device=dev)
        qidx = torch.from_numpy(mine).to(dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        L.check(L.lib.grab_shard_pack(len(mine), L.ptr(qidx), L.ptr(slots.contiguous()), L.ptr(dists.contiguous()),
                                      L.ptr(self.gid), k, self.world, B, L.ptr(send_d), L.ptr(send_i), stream))
        recv_d, recv_i = exchange(send_d, send_i, self.world, self.group, self.device)
        first = self.rank * B
        n_own = max(0, min(B, nq - first))
        out_d = torch.empty((n_own, k), dtype=torch.float64, device=dev)
        out_i = torch.empty((n_own, k), dtype=torch.int64, device=dev)
        out_c = torch.empty(n_own, dtype=torch.int32, device=dev)
        L.check(L.lib.grab_merge_topk(n_own, self.world, B, k, L.ptr(recv_d), L.ptr(recv_i), L.ptr(out_d),
                                      L.ptr(out_i), L.ptr(out_c), torch.cuda.current_stream(dev).cuda_stream))
        return ShardResult(first, out_i, out_d, out_c, len(mine))


def _coll_device(group, device):
    """Device for collective tensors: CUDA under NCCL, CPU under gloo."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group) if dist.is_initialized() else "none"
    return torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")


def exchange(send_d, send_i, world: int, group=None, device: int = 0):
    """Fixed-size all-to-all of the per-owner blocks [world, B, k]: block r of
    every rank lands at recv[src] on rank r. NCCL moves device memory over
    NVLink; gloo (CPU tests) stages through the host."""
    if world == 1:
        return send_d, send_i
    import torch
    import torch.distributed as dist
    cdev = _coll_device(group, device)
    out = []
    for t in (send_d, send_i):
        src = t.to(cdev)
        dst = torch.empty_like(src)
        dist.all_to_all_single(dst, src, group=group)
        out.append(dst.to(t.device))
    return out[0], out[1]


def merge_reference(recv_d: np.ndarray, recv_i: np.ndarray, n_own: int, k: int):
    """Host restatement of grab_merge_topk for the tests: per owned query, the
    k smallest (distance, id) over the world lists (entries with id < 0 empty)."""
    world = recv_d.shape[0]
    slots = np.full((n_own, k), -1, dtype=np.int64)
    dists = np.full((n_own, k), np.nan)
    counts = np.zeros(n_own, dtype=np.int64)
    for q in range(n_own):
        cand = [(recv_d[r, q, j], recv_i[r, q, j]) for r in range(world) for j in range(k) if recv_i[r, q, j] >= 0]
        cand.sort()
        cand = cand[:k]
        counts[q] = len(cand)
        for j, (d, i) in enumerate(cand):
            slots[q, j] = i
            dists[q, j] = d
    return slots, dists, counts
