"""Two ranks on the GPU box (both on cuda:0, gloo for the collective since one
device cannot host two NCCL ranks): real kernels, real doc sharding, real
all-reduce of the device phi-count buffer through distributed.ShardedTrainer.
The sharded phi must equal single-process training bit for bit -- the
property the NCCL run on 8 B200s relies on.  On a box with >= 2 GPUs the same
test runs one rank per GPU over NCCL (the production path, device buffers
reduced in place)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

K, SEED, M, T_MAX, BF = 8, 7, 20.0, 5, 0.25


def _corpus():
    from oracle import Port
    port = Port()
    return port.make_corpus(120, 60, 4, 30.0, 3)


def _worker(rank, world, port_no, out_path, mode=0, backend="gloo", engine_kind="host"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1409_5402_b200 import distributed as D
    from paper_1409_5402_b200 import samelda as S
    g = _corpus()
    lo, hi = D.shard_ranges(g.doc_offsets, world)[rank]
    offs = g.doc_offsets[lo:hi + 1] - g.doc_offsets[lo]
    local = S.Corpus(offs, g.word_ids[g.doc_offsets[lo]:g.doc_offsets[hi]],
                     g.counts[g.doc_offsets[lo]:g.doc_offsets[hi]], g.n_words)
    ctx = S.Context(dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    cfg = S.SamplerConfig(n_topics=K, m=M, schedule="invlinear", t_max=T_MAX, batch_fraction=BF,
                          seed=SEED, mode=mode)
    tr = S.Trainer(local, cfg, ctx=ctx)

    class GlooEngine(D.CudaEngine):
        """gloo reduces host tensors: stage the device counts through the host
        (the plain u64 all-reduce, no int32 packing)."""

        exchange = None

        def counts(self):
            self._host = super().counts().cpu()
            return self._host

        def update(self, rho):
            super().counts().copy_(self._host)
            super().update(rho)

    # engine_kind "device": the production engine (int32 count exchange of
    # device tensors), here over gloo's CUDA all-reduce
    engine = GlooEngine(tr, 0) if backend == "gloo" and engine_kind == "host" else D.CudaEngine(tr, dev)
    # ShardedTrainer sets the engine's doc base (global Philox doc ids)
    st = D.ShardedTrainer(engine, g.n_docs, lo, hi, local.doc_tokens(), BF, SEED, M,
                          "invlinear", T_MAX)
    for _ in range(T_MAX):
        st.period()
    model = tr.model()
    if rank == 0:
        np.savez(out_path, phi=model.phi, theta_rows=model.theta)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(600)
@pytest.mark.parametrize("mode", [0, 2], ids=["parity", "throughput"])
def test_two_rank_sharded_training_equals_single_gpu(tmp_path, mode):
    """Both modes key their streams by global document ids and scatter
    integer counts, so the sharded result is the single-GPU result bit for
    bit (the throughput mode's own streams included)."""
    from paper_1409_5402_b200 import samelda as S
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out, mode), nprocs=2, start_method="spawn")
    got = np.load(out)
    g = _corpus()
    model, _ = S.train(g, S.SamplerConfig(n_topics=K, m=M, schedule="invlinear", t_max=T_MAX,
                                          batch_fraction=BF, seed=SEED, mode=mode))
    np.testing.assert_array_equal(got["phi"], model.phi)


@pytest.mark.timeout(600)
def test_two_rank_int32_exchange_equals_single_gpu(tmp_path):
    """The production engine's count exchange in int32 words (pack32 on the
    device, the 8-byte over-bound count all-reduced first, the packed words
    all-reduced and unpacked in place) leaves phi bit-equal to one GPU."""
    from paper_1409_5402_b200 import samelda as S
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out, 0, "gloo", "device"), nprocs=2,
                       start_method="spawn")
    got = np.load(out)
    model, _ = S.train(_corpus(), S.SamplerConfig(n_topics=K, m=M, schedule="invlinear",
                                                  t_max=T_MAX, batch_fraction=BF, seed=SEED))
    np.testing.assert_array_equal(got["phi"], model.phi)


def test_pack32_unpack32_roundtrip_and_bound():
    """pack32 copies every count below (2^31 - 1) / world_size exactly and counts
    the cells at or above it; unpack32 writes int32 words back as u64 counts."""
    from paper_1409_5402_b200 import distributed as D
    from paper_1409_5402_b200 import samelda as S
    g = _corpus()
    ctx = S.Context(0)
    stream = torch.cuda.Stream(device=0)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    tr = S.Trainer(g, S.SamplerConfig(n_topics=K, m=M, t_max=2, batch_fraction=1.0, seed=SEED), ctx=ctx)
    eng = D.CudaEngine(tr, 0)
    tr.period_sample(np.arange(g.n_docs, dtype=np.int32), 1, M)
    c = eng.counts()
    ref = c.clone()
    n = c.numel()
    lo = torch.empty(n, dtype=torch.int32, device="cuda:0")
    over = torch.zeros(1, dtype=torch.int64, device="cuda:0")
    tr.phi_counts_pack32(lo.data_ptr(), n, 8, over.data_ptr())
    torch.cuda.synchronize()
    assert int(over.item()) == 0 and int(ref.sum()) > 0
    assert torch.equal(lo.to(torch.int64), ref)
    # a bound of (2^31 - 1) // 2^30 = 1: every nonzero cell is over it
    tr.phi_counts_pack32(lo.data_ptr(), n, 2**30, over.data_ptr())
    torch.cuda.synchronize()
    assert int(over.item()) == int((ref >= 1).sum())
    lo2 = (lo * 3).contiguous()
    torch.cuda.synchronize()
    tr.phi_counts_unpack32(lo2.data_ptr(), n)
    torch.cuda.synchronize()
    assert torch.equal(eng.counts(), ref * 3)


def test_bench_two_rank_path_runs(tmp_path):
    """bench.py's torchrun path (N=2, weak scaling, one global minibatch
    stream, per-period count all-reduce) end to end on the one-GPU box
    (BENCH_SHARE_GPU: both ranks on cuda:0 over gloo); the JSON line is
    well-formed and reports the aggregate over ranks."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BENCH_SHARE_GPU="1", BENCH_NO_CLOCKS="1")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(port_no), "bench.py", "--gpus", "2",
         "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--scaling", "weak"],
        cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["parallelism"] == "doc-shard x2" and line["scaling"] == "weak"


@pytest.mark.timeout(600)
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (NCCL ranks)")
@pytest.mark.parametrize("mode", [0, 2], ids=["parity", "throughput"])
def test_nccl_ranks_equal_single_gpu(tmp_path, mode):
    """One rank per GPU over NCCL (the bench's multi-GPU path): phi bit-equal to one GPU."""
    from paper_1409_5402_b200 import samelda as S
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out, mode, "nccl"), nprocs=2,
                       start_method="spawn")
    got = np.load(out)
    model, _ = S.train(_corpus(), S.SamplerConfig(n_topics=K, m=M, schedule="invlinear",
                                                  t_max=T_MAX, batch_fraction=BF, seed=SEED,
                                                  mode=mode))
    np.testing.assert_array_equal(got["phi"], model.phi)


def test_bench_launches_its_own_ranks():
    """`python bench.py --gpus 2` outside torchrun re-launches itself with one process per
    rank (here both on cuda:0 over gloo: BENCH_SHARE_GPU) on the stated corpus, strong
    scaling: the line reports n_gpus 2 and doc-shard x2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(BENCH_SHARE_GPU="1", BENCH_NO_CLOCKS="1")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup",
                          "3", "--no-cpu-baseline"], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["parallelism"] == "doc-shard x2"
    assert line["corpus"]["train_docs"] == 270000 and line["value"] > 0
