"""Document-sharded SAME training across ranks (one process per GPU).

Documents are independent given phi, so rank r owns a
contiguous range of documents -- their CSR rows, theta rows and theta counts.
Every rank runs the same global MinibatchStream (corpus.cpp:252-285) and
samples only the batch documents it owns; Philox keys use the GLOBAL doc id
(`samelda_cu_set_doc_base`), so each rank draws exactly what one GPU would.
The one exchange per period is a sum all-reduce of the W x K topic-word
counts of the last inner sweep (sampler.cpp:320-332).  In the integer-count
modes (parity, throughput) addition is associative, so the reduced counts --
and the replicated M-step's phi -- are bit-identical to a single-GPU run; the
expected-count mode all-reduces f64 sums, whose order (and so last bits) the
collective chooses.

`torch.distributed` is the plumbing (NCCL on B200s, gloo in the CPU tests);
the per-rank compute is an *engine*: `CudaEngine` (the product, over
libsamelda_cuda.so) or a test engine built on the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np


def shard_ranges(doc_offsets: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous doc ranges balanced by nonzeros (parallel.hpp:29-43's idea)."""
    doc_offsets = np.asarray(doc_offsets, np.int64)
    D = len(doc_offsets) - 1
    total = int(doc_offsets[-1])
    bounds = [0]
    for i in range(1, world):
        target = total * i // world
        pos = int(np.searchsorted(doc_offsets[:D], target, side="left"))
        bounds.append(max(bounds[-1], min(pos, D)))
    bounds.append(D)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def owned(batch: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Batch docs in [lo, hi) as local ids, batch order preserved."""
    batch = np.asarray(batch)
    sel = batch[(batch >= lo) & (batch < hi)]
    return (sel - lo).astype(np.int32)


class _CAI:
    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 2, "strides": None}


class CudaEngine:
    """Per-rank engine over the device-resident trainer (samelda.Trainer)."""

    def __init__(self, trainer, device: int):
        import torch
        self.trainer = trainer
        self.device = device
        self._counts = None
        self._lo = self._over = None
        # the count all-reduce is enqueued on torch's current stream: run the
        # trainer on that stream so the collective is ordered after sampling
        trainer.ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)

    def set_doc_base(self, base: int):
        self.trainer.set_doc_base(base)

    def sample(self, local_ids, t, m_t):
        self.trainer.period_sample(local_ids, t, m_t)

    def counts(self):
        if self._counts is None:
            import torch
            ptr, n, _, is_f = self.trainer.phi_counts_device()
            self._counts = torch.as_tensor(_CAI(ptr, n, "<f8" if is_f else "<i8"),
                                           device=f"cuda:{self.device}")
        return self._counts

    def exchange(self, group=None):
        """The per-period all-reduce of the W x K counts.  Integer counts go
        as int32 words (half the bytes): packed on the device, the number of
        cells too large for an exact int32 sum over the ranks all-reduced
        first (8 bytes), then either the packed words (unpacked in place) or,
        if any rank had such a cell, the untouched u64 counts.  Expected-mode
        f64 counts are all-reduced as they are."""
        import torch
        import torch.distributed as dist
        counts = self.counts()
        if counts.dtype != torch.int64 or os.environ.get("SAMELDA_EXCHANGE") == "u64":
            dist.all_reduce(counts, group=group)
            return
        n = counts.numel()
        if self._lo is None or self._lo.numel() != n:
            self._lo = torch.empty(n, dtype=torch.int32, device=counts.device)
            self._over = torch.zeros(1, dtype=torch.int64, device=counts.device)
        self.trainer.phi_counts_pack32(self._lo.data_ptr(), n, dist.get_world_size(group),
                                       self._over.data_ptr())
        dist.all_reduce(self._over, group=group)
        if int(self._over.item()) == 0:  # the one host wait of the exchange
            dist.all_reduce(self._lo, group=group)
            self.trainer.phi_counts_unpack32(self._lo.data_ptr(), n)
        else:
            dist.all_reduce(counts, group=group)

    def update(self, rho_t):
        self.trainer.period_update(rho_t)


@dataclass
class PeriodStats:
    t: int
    m_t: float
    rho_t: float
    batch_docs: int
    owned_docs: int
    owned_tokens: float


class ShardedTrainer:
    """The train() period loop (sampler.cpp:307-339) over doc shards."""

    def __init__(self, engine, n_docs_global: int, doc_lo: int, doc_hi: int,
                 local_doc_tokens: np.ndarray, batch_fraction: float, seed: int, m: float,
                 schedule: str, t_max: int, tau0: float = 1.0, gamma: float = 0.5,
                 group=None):
        from . import samelda as S
        self.S = S
        self.engine = engine
        self.lo, self.hi = doc_lo, doc_hi
        self.doc_tokens = np.asarray(local_doc_tokens, np.float64)
        self.batches = S.MinibatchStream(n_docs_global, batch_fraction, seed)
        self.m, self.schedule, self.t_max = m, schedule, t_max
        self.tau0, self.gamma = tau0, gamma
        self.group = group
        self.t = 0
        # Philox keys use GLOBAL doc ids: the engine's local doc 0 is global
        # doc_lo (an engine without the hook keys streams itself, e.g. a test
        # engine that receives global ids)
        if hasattr(engine, "set_doc_base"):
            engine.set_doc_base(doc_lo)

    def period(self) -> PeriodStats:
        import torch.distributed as dist
        t = self.t
        batch = self.batches.next()
        own = owned(batch, self.lo, self.hi)
        m_t = self.S.anneal_m(self.schedule, t + 1, self.t_max, self.m)
        rho = self.S.rho_schedule(t, self.tau0, self.gamma)
        self.engine.sample(own, t, m_t)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            exchange = getattr(self.engine, "exchange", None)
            if exchange is not None:
                exchange(self.group)
            else:
                dist.all_reduce(self.engine.counts(), group=self.group)
        self.engine.update(rho)
        self.t += 1
        return PeriodStats(t, m_t, rho, len(batch), len(own), float(self.doc_tokens[own].sum()))
