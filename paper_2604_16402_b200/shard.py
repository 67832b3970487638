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
   the CPU tests) -- or, with ``exchange="p2p"``, no collective at all: the pack
   kernel stores straight into each owner's receive buffer through CUDA IPC
   mappings (NVLink peer memory), bracketed by two barriers;
5. ``grab_merge_topk``: each owner merges world x k candidates per query by
   (distance, global id), the reference's tie rule.

No query is replicated beyond the routing and no shard scans rows outside its
range; cross-shard edges do not exist (each shard is an independent graph), so
recall is measured against the global exact oracle (the same pipeline with the
brute-force kernel in step 2).
"""
from __future__ import annotations

import ctypes as C
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

    def __init__(self, local, gid, spans: np.ndarray, rank: int, world: int, group=None, device: int = 0,
                 exchange: str = "nccl"):
        import torch
        if exchange not in ("nccl", "p2p"):
            raise ValueError(f"unknown exchange: {exchange!r}")
        self.local = local
        self.rank, self.world, self.group, self.device = rank, world, group, device
        self.exchange = exchange
        self.spans = np.asarray(spans, dtype=np.float32)
        self.gid = torch.as_tensor(np.ascontiguousarray(gid, dtype=np.int64), device=self._dev())
        self._peers = None  # (B, k) -> peer receive buffers for exchange="p2p"

    def _peer_buffers(self, B: int, k: int):
        """Receive buffers [world][B][k] (dists, ids) on every rank, mapped into
        every other rank through CUDA IPC (allocated once per (B, k))."""
        import torch
        import torch.distributed as dist
        if self._peers is not None and self._peers["shape"] == (B, k):
            return self._peers
        if self._peers is not None and self.world > 1:
            # (setup, not per batch) every rank is past its last merge before
            # the old buffers go away
            torch.cuda.current_stream(self._dev()).synchronize()
            dist.barrier(group=self.group)
        self.close_peers()
        nbytes = self.world * B * k * 8
        own, handles = [], []
        # receive buffers (dists, ids) and the sync block of the device-side flags
        # (grab_ipc_alloc zero-fills: the sync block starts at epoch 0 -- every
        # buffer free, nothing ready)
        for nb in (nbytes, nbytes, int(L.lib.grab_shard_sync_bytes(self.world))):
            p = C.c_void_p()
            h = (C.c_uint8 * 64)()
            L.check(L.lib.grab_ipc_alloc(nb, C.byref(p), h))
            own.append(p.value)
            handles.append(bytes(h))
        if self.world > 1:
            allh = [None] * self.world
            dist.all_gather_object(allh, handles, group=self.group)
        else:
            allh = [handles]
        ptrs, opened = [[0] * self.world, [0] * self.world, [0] * self.world], []
        for r in range(self.world):
            for t in range(3):
                if r == self.rank:
                    ptrs[t][r] = own[t]
                else:
                    p = C.c_void_p()
                    hb = (C.c_uint8 * 64).from_buffer_copy(allh[r][t])
                    L.check(L.lib.grab_ipc_open(hb, C.byref(p)))
                    ptrs[t][r] = p.value
                    opened.append(p.value)
        dev = self._dev()
        self._peers = {"shape": (B, k), "own": own, "opened": opened,
                       "ptr_d": torch.tensor(ptrs[0], dtype=torch.int64, device=dev),
                       "ptr_i": torch.tensor(ptrs[1], dtype=torch.int64, device=dev),
                       "ptr_sync": torch.tensor(ptrs[2], dtype=torch.int64, device=dev), "epoch": 0,
                       "inv": torch.empty(self.world * B, dtype=torch.int32, device=dev)}
        if self.world > 1:
            dist.barrier(group=self.group)  # every rank zeroed its sync block before any pack runs
        return self._peers

    def close_peers(self) -> None:
        if self._peers is None:
            return
        for p in self._peers["opened"]:
            L.lib.grab_ipc_close(C.c_void_p(p))
        for p in self._peers["own"]:
            L.lib.grab_ipc_free(C.c_void_p(p))
        self._peers = None

    def _dev(self):
        import torch
        return torch.device("cuda", self.device)

    # ------------------------------------------------------------------ build
    @classmethod
    def build(cls, X_local, S_local, gid_local, params: BuildParams, *, rank: int, world: int, group=None,
              device: int = 0, exchange: str = "nccl", **build_kw):
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
        return cls(local, gid_local, spans, rank, world, group, device, exchange), report

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
        qidx = torch.from_numpy(mine).to(dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        if self.exchange == "p2p":
            # fused exchange: stores straight into the owners' receive buffers over
            # NVLink, ordered by device-side peer flags (epoch per batch): the host
            # enqueues search -> pack -> merge and never waits
            pb = self._peer_buffers(B, k)
            pb["epoch"] += 1
            L.check(L.lib.grab_shard_pack_p2p_sync(nq, len(mine), L.ptr(qidx), L.ptr(slots.contiguous()),
                                                   L.ptr(dists.contiguous()), L.ptr(self.gid), k, self.rank,
                                                   self.world, B, L.ptr(pb["ptr_d"]), L.ptr(pb["ptr_i"]),
                                                   C.c_void_p(pb["own"][2]), L.ptr(pb["ptr_sync"]), pb["epoch"],
                                                   L.ptr(pb["inv"]), stream))
            recv_d, recv_i = C.c_void_p(pb["own"][0]), C.c_void_p(pb["own"][1])
        else:
            send_d = torch.empty((self.world, B, k), dtype=torch.float64, device=dev)
            send_i = torch.empty((self.world, B, k), dtype=torch.int64, device=dev)
            L.check(L.lib.grab_shard_pack(len(mine), L.ptr(qidx), L.ptr(slots.contiguous()),
                                          L.ptr(dists.contiguous()), L.ptr(self.gid), k, self.world, B,
                                          L.ptr(send_d), L.ptr(send_i), stream))
            recv_d, recv_i = exchange(send_d, send_i, self.world, self.group, self.device)
        first = self.rank * B
        n_own = max(0, min(B, nq - first))
        out_d = torch.empty((n_own, k), dtype=torch.float64, device=dev)
        out_i = torch.empty((n_own, k), dtype=torch.int64, device=dev)
        out_c = torch.empty(n_own, dtype=torch.int32, device=dev)
        rd = recv_d if isinstance(recv_d, C.c_void_p) else L.ptr(recv_d)
        ri = recv_i if isinstance(recv_i, C.c_void_p) else L.ptr(recv_i)
        if self.exchange == "p2p":
            L.check(L.lib.grab_merge_topk_p2p(n_own, self.world, B, k, rd, ri, L.ptr(out_d), L.ptr(out_i),
                                              L.ptr(out_c), self.rank, C.c_void_p(pb["own"][2]),
                                              L.ptr(pb["ptr_sync"]), pb["epoch"], stream))
        else:
            L.check(L.lib.grab_merge_topk(n_own, self.world, B, k, rd, ri, L.ptr(out_d),
                                          L.ptr(out_i), L.ptr(out_c), stream))
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
