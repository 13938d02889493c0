"""Request-stream serving across GPUs (config 5; BASELINE.json north_star: "a stream of
variable-length inference requests is partitioned across the 8 GPUs of one box, each
GPU running whole requests with no collectives beyond an NCCL gather of results").

* shard():  deterministic LPT partition of the request list (nimble_partition_lpt,
  native) — every rank computes the same partition, no communication.
* GraphCache: one CUDA graph per distinct sequence length L, captured once (the
  dynamic kernels + their dispatch decisions for that L; capture = Nimble's
  "compile once, dispatch at run time", replay = the launch-overhead-free VM
  InvokePacked stream).  Shape functions and dispatch still run at capture time
  through the C ABI for each L.
* gather_results(): the one collective — a padded torch.distributed gather of
  (request id, [CLS] vector) to rank 0 (NCCL over NVLink on the GPU box; gloo in
  the CPU tests).  Rank 0 reorders by request id.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import nimble as nb


def shard(lens: np.ndarray, world: int, rank: int) -> np.ndarray:
    """Request ids owned by `rank` (ascending), from the native LPT partition."""
    owner = nb.partition_lpt(lens, world)
    return np.nonzero(owner == rank)[0].astype(np.int64)


class GraphCache:
    """Per-L CUDA graphs of a full encoder forward for ONE request (batch 1), reading a static
    input buffer and writing the [CLS] row into a static output row.  The encoder is either a
    BertPacked over a single request (7 launches per layer, fused attention) or a BertEncoder
    (9 launches per layer: bmm_dyn -> softmax -> bmm_dyn attention)."""

    def __init__(self, encoder, device="cuda"):
        self.enc = encoder
        self.packed = hasattr(encoder, "max_tokens")
        max_len = encoder.max_tokens if self.packed else encoder.max_len
        self.xin = torch.zeros((max_len, encoder.d), dtype=torch.bfloat16, device=device)
        self.cls = torch.zeros((encoder.d,), dtype=torch.bfloat16, device=device)
        self.offs = {}
        self.graphs = {}
        self.stream = torch.cuda.Stream(device=device)

    def _forward(self, L: int):
        if self.packed:
            if L not in self.offs:                  # created before capture (no H2D inside a graph)
                self.offs[L] = torch.tensor([0, L], dtype=torch.int32, device=self.xin.device)
            return self.enc.forward(self.xin, self.offs[L], L, T=L)
        return self.enc.forward(self.xin, L)

    def capture(self, L: int):
        if L in self.graphs:
            return
        g = torch.cuda.CUDAGraph()
        s = self.stream
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._forward(L)                       # warm (lazy attribute setup) outside capture
            with torch.cuda.graph(g, stream=s):
                y = self._forward(L)
                self.cls.copy_(y[0])
        torch.cuda.current_stream().wait_stream(s)
        self.graphs[L] = g

    def capture_all(self, lengths):
        for L in sorted(set(int(x) for x in lengths)):
            self.capture(L)

    def run(self, x: torch.Tensor, L: int, out_row: torch.Tensor):
        """x [L x d] device; out_row [d] device receives the [CLS] vector (stream-ordered)."""
        self.xin[:L].copy_(x, non_blocking=True)
        self.graphs[L].replay()
        out_row.copy_(self.cls, non_blocking=True)


class DeviceExtentGraph:
    """ONE CUDA graph of the one-request packed forward whose token count lives on the device
    (BertPacked.forward_dev: device-side dispatch, extent-patched tensor maps; SURVEY §8 f4 /
    PAPER.md:268-271, 709-710).  It replays for every L <= max_tokens (< 2048): no per-L
    capture, no per-L graph memory.  Same interface as GraphCache."""

    def __init__(self, encoder, device="cuda"):
        assert hasattr(encoder, "forward_dev") and encoder.max_tokens < 2048
        self.enc = encoder
        Tm = encoder.max_tokens
        self.xin = torch.zeros((Tm, encoder.d), dtype=torch.bfloat16, device=device)
        self.cls = torch.zeros((encoder.d,), dtype=torch.bfloat16, device=device)
        self.seq_off = torch.tensor([0, Tm], dtype=torch.int32, device=device)
        self.stream = torch.cuda.Stream(device=device)
        self.graph = torch.cuda.CUDAGraph()
        s = self.stream
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            encoder.forward_dev(self.xin, self.seq_off)          # warm outside capture
            with torch.cuda.graph(self.graph, stream=s):
                y = encoder.forward_dev(self.xin, self.seq_off)
                self.cls.copy_(y[0])
        torch.cuda.current_stream().wait_stream(s)

    def capture(self, L: int):             # nothing to do: one graph serves every L
        assert 1 <= L <= self.enc.max_tokens

    def capture_all(self, lengths):
        for L in lengths:
            self.capture(int(L))

    def run(self, x: torch.Tensor, L: int, out_row: torch.Tensor):
        self.xin[:L].copy_(x, non_blocking=True)
        self.seq_off[1:].fill_(L)          # the extent, written on the stream (no host sync)
        self.graph.replay()
        out_row.copy_(self.cls, non_blocking=True)


def run_requests(cache: GraphCache, ids, lens, X_all: torch.Tensor, offsets, out: torch.Tensor):
    """Run whole requests (batch 1 each) in id order; out[i] = [CLS] of request ids[i]."""
    for i, rid in enumerate(ids):
        L = int(lens[rid])
        o = int(offsets[rid])
        cache.run(X_all[o:o + L], L, out[i])


class ResultGather:
    """The one collective of the request-sharded stream (§8(e)): every step, each rank's
    (request id, [CLS]) rows are gathered to rank 0 into preallocated buffers, with no host
    synchronisation (the ids are padded to max_count with -1; nothing is compacted on the
    hot path).  `result()` — called once, after the timed region — drops the padding and
    orders rank 0's rows by request id."""

    def __init__(self, max_count: int, d: int, world: int, rank: int, device, dtype=torch.bfloat16):
        self.world, self.rank, self.max_count = world, rank, max_count
        self.ids_pad = torch.full((max_count,), -1, dtype=torch.int64, device=device)
        self.cls_pad = torch.zeros((max_count, d), dtype=dtype, device=device)
        if world > 1 and rank == 0:
            self.all_ids = [torch.empty_like(self.ids_pad) for _ in range(world)]
            self.all_cls = [torch.empty_like(self.cls_pad) for _ in range(world)]
        else:
            self.all_ids = [self.ids_pad] if world == 1 else None
            self.all_cls = [self.cls_pad] if world == 1 else None

    def step(self, ids_local: torch.Tensor, cls_local: torch.Tensor):
        n = ids_local.shape[0]
        if n:
            self.ids_pad[:n].copy_(ids_local, non_blocking=True)
            self.cls_pad[:n].copy_(cls_local, non_blocking=True)
        if self.world > 1:
            dist.gather(self.ids_pad, self.all_ids, dst=0)
            dist.gather(self.cls_pad, self.all_cls, dst=0)

    def result(self):
        """(ids, cls) sorted by id on rank 0 (padding dropped); (None, None) elsewhere."""
        if self.rank != 0:
            return None, None
        ids = torch.cat(self.all_ids)
        cls = torch.cat(self.all_cls)
        keep = ids >= 0
        ids, cls = ids[keep], cls[keep]
        order = torch.argsort(ids)
        return ids[order], cls[order]


def gather_results(ids_local: torch.Tensor, cls_local: torch.Tensor, max_count: int, world: int, rank: int):
    """One-shot form of ResultGather: gather (ids, [CLS]) from every rank to rank 0; returns
    (ids, cls) sorted by id on rank 0, (None, None) elsewhere."""
    g = ResultGather(max_count, cls_local.shape[1], world, rank, cls_local.device, cls_local.dtype)
    g.step(ids_local, cls_local)
    return g.result()
