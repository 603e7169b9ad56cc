"""SAME factored Gibbs sampler benchmark (BASELINE.json metric and configs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config nytimes|c1|c3|pubmed|k1024|nytimes-expected|nytimes-fast]
                    [--scaling strong|weak]

A step is one SAME period (Algorithm 3; sampler.cpp:307-333) over one
minibatch of the synthetic corpus: inner_sweeps x (SDDMM + Poisson replica
sampling + count scatter) and the M-step.  Metric: sampled token x replica
samples per second = sum over sweeps of (batch tokens x m_t) / time.

Configs (BASELINE.json `configs`):
  c1       [0] the reference's own synthetic corpus make_corpus(10000, 5000, 32, 100, 1),
               split_holdout(0.1, 1), K=32, m=10, full-batch periods, eval every 5;
               e2e = the whole 20-period train() through the C ABI (samelda_cu_train)
               against the reference's train() on the host cores
  nytimes  [1] (default) NYTimes-shaped synthetic corpus (300K docs, 102,660 words,
               ~100M tokens, ~70M nonzeros), K=256, m=100, bf=0.05, 2 inner sweeps
  c3       [2] the same corpus with the linear annealing schedule: m_t = 2 m t / (T+1),
               m = 50, T = the periods of the run, so m_t rises from ~1 to ~100
  pubmed   [3] PubMed-shaped synthetic corpus (8.2M docs, 141,043 words, ~730M tokens)
  k1024    [4] the NYTimes corpus at K=1024, m=50
  nytimes-expected / nytimes-fast: the deterministic expected-count path and the
               throughput mode on config [1]

Multi-GPU: `--gpus N` with N > 1 outside torchrun re-launches this script
under `torch.distributed.run` (one process per GPU, NCCL; 127.0.0.1).
Strong scaling (default): the config's corpus is split into N contiguous
document ranges, each rank generates and holds only its own; all ranks run
one global MinibatchStream, each samples the batch docs it owns (Philox keys
use global doc ids, so the draws equal one GPU's), the W x K topic-word
counts are all-reduced over NCCL once per period, the M-step is replicated.
`--scaling weak`: every rank holds its own full-size shard (N x the corpus).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sampled tokens/sec (x m replicas)"

CONFIGS = {
    "c1": dict(baseline=0, corpus="c1", n_topics=32, m=10.0, batch_fraction=1.0, inner_sweeps=2,
               schedule="constant", t_max=20, eval_every=5,
               workload="reference synthetic corpus make_corpus(10000 docs, 5000 words, 32 topics, "
                        "len 100, seed 1) split_holdout(0.1, 1), K=32, m=10, full-batch periods "
                        "(20 iterations), 2 inner sweeps, eval every 5"),
    "nytimes": dict(baseline=1, corpus="nytimes", n_topics=256, m=100.0, batch_fraction=0.05,
                    inner_sweeps=2, schedule="constant",
                    workload="NYTimes-shaped synthetic corpus (300K docs, 102,660 vocab, ~100M "
                             "tokens), K=256, m=100, bf=0.05, 2 inner sweeps"),
    "c3": dict(baseline=2, corpus="nytimes", n_topics=256, m=50.0, batch_fraction=0.05,
               inner_sweeps=2, schedule="linear",
               workload="NYTimes-shaped synthetic corpus, K=256, SAME annealing m_t = 2*50*t/(T+1) "
                        "(~1 to ~100 over the run's T periods), bf=0.05, 2 inner sweeps"),
    "pubmed": dict(baseline=3, corpus="pubmed", n_topics=256, m=100.0, batch_fraction=0.05,
                   inner_sweeps=2, schedule="constant",
                   workload="PubMed-shaped synthetic corpus (8.2M docs, 141,043 vocab, ~730M "
                            "tokens), K=256, m=100, bf=0.05"),
    "k1024": dict(baseline=4, corpus="nytimes", n_topics=1024, m=50.0, batch_fraction=0.05,
                  inner_sweeps=2, schedule="constant",
                  workload="NYTimes-shaped synthetic corpus, K=1024, m=50, bf=0.05"),
    "nytimes-expected": dict(baseline=1, corpus="nytimes", n_topics=256, m=100.0,
                             batch_fraction=0.05, inner_sweeps=2, schedule="constant",
                             mode="expected",
                             workload="NYTimes-shaped synthetic corpus, K=256, m=100, bf=0.05, "
                                      "2 inner sweeps, expected-count mode"),
    "nytimes-fast": dict(baseline=1, corpus="nytimes", n_topics=256, m=100.0, batch_fraction=0.05,
                         inner_sweeps=2, schedule="constant", mode="throughput",
                         workload="NYTimes-shaped synthetic corpus, K=256, m=100, bf=0.05, "
                                  "2 inner sweeps, throughput mode (f32, own random streams)"),
    "nytimes-multinomial": dict(baseline=1, corpus="nytimes", n_topics=256, m=100.0,
                                batch_fraction=0.05, inner_sweeps=2, schedule="constant",
                                mode="multinomial",
                                workload="NYTimes-shaped synthetic corpus, K=256, m=100, bf=0.05, "
                                         "2 inner sweeps, multinomial(c m) replicas (own streams)"),
    "nytimes-converged": dict(baseline=1, corpus="nytimes", n_topics=256, m=100.0,
                              batch_fraction=0.05, inner_sweeps=2, schedule="constant",
                              pre_periods=100,
                              workload="NYTimes-shaped synthetic corpus, K=256, m=100, bf=0.05, "
                                       "2 inner sweeps, timed after 100 untimed periods (5 passes: "
                                       "a converged model, nearly every nonzero with a PTRS draw)"),
}
ALIASES = {"c2": "nytimes", "c4": "pubmed", "c5": "k1024"}

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        if os.environ.get("BENCH_NO_CLOCKS"):
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self._t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ setup

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch_under_torchrun(n: int) -> int:
    """One process per GPU: re-exec this script under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    # NCCL communicator setup in the log (rank count per communicator)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=env, cwd=ROOT).returncode


class Workload:
    """The config's corpus as seen by one rank: its training documents (a contiguous range
    [doc_lo, doc_lo + D_local) of the global training corpus), the held-out corpus (rank 0),
    and the global sizes every arm reports."""

    def __init__(self, cfg, world: int, rank: int, scaling: str):
        from paper_1409_5402_b200 import synth
        t0 = time.perf_counter()
        self.world, self.rank = world, rank
        if cfg["corpus"] == "c1":
            whole = synth.make_corpus_ref(10000, 5000, 32, 100.0, 1)
            train, test = synth.split_holdout(whole, 0.1, 1)  # commands.cpp:89-90
            self.D_global = train.n_docs
            lo, hi = train.n_docs * rank // world, train.n_docs * (rank + 1) // world
            self.train = synth.subset(train, np.arange(lo, hi)) if world > 1 else train
            self.doc_lo = lo
            self.heldout = test if rank == 0 else None
            self.total_docs = whole.n_docs
        else:
            kw = dict(synth.PRESETS[cfg["corpus"]])
            D = kw.pop("n_docs")
            n_test = max(1, int(round(0.1 * D)))  # the last 10% of the (iid) docs are held out
            cut = D - n_test
            if scaling == "weak":  # rank r: global docs [r D, (r + 1) D), its own full shard
                first, lo, hi = rank * D, 0, cut
                self.D_global = cut * world
                self.doc_lo = rank * cut
                self.total_docs = D * world
            else:  # strong: the one corpus, training docs split into N contiguous ranges
                first = 0
                lo, hi = cut * rank // world, cut * (rank + 1) // world
                self.D_global = cut
                self.doc_lo = lo
                self.total_docs = D
            self.train = synth.generate(seed=1, n_docs=hi - lo, first_doc=first + lo, **kw)
            self.heldout = (synth.generate(seed=1, n_docs=n_test, first_doc=first + cut, **kw)
                            if rank == 0 else None)
        self.gen_s = time.perf_counter() - t0


def single_gpu_corpus(config: str = "nytimes"):
    """(train, heldout) of a config's corpus as one GPU holds it (tests, tools)."""
    wl = Workload(CONFIGS[ALIASES.get(config, config)], 1, 0, "strong")
    return wl.train, wl.heldout


# --------------------------------------------------------- shared record

def config_record(cfg, world: int, scaling: str) -> dict:
    """The `config` object -- identical in both arms for the same command line."""
    return {"workload": cfg["workload"], "baseline_config": cfg["baseline"],
            "K": cfg["n_topics"], "m": cfg["m"], "schedule": cfg["schedule"],
            "batch_fraction": cfg["batch_fraction"], "inner_sweeps": cfg["inner_sweeps"],
            "mode": cfg.get("mode", "parity"), "parallelism": f"doc-shard x{world}",
            "scaling": scaling,
            "l2": "inputs larger than L2 (phi + theta resident in HBM; random minibatch docs "
                  "each step)" if cfg["corpus"] != "c1" else
                  "C1 model (phi 1.3 MB) is L2-resident by design"}


# the end-to-end leg runs this many times back to back (best reported, every
# leg's value listed): a one-off ~0.1 s host stall inside one ~70 ms leg (seen
# on some runs, from the host side: no device gap) would otherwise decide it
E2E_LEGS = 3


def run_t_max(cfg, args) -> int:
    """Periods the run performs (warm-up, timed, profiled, end-to-end over as many
    periods as the timed region): the annealing schedule's horizon T (c3: m_t rises
    over exactly this run)."""
    prof = max(1, min(args.steps, 10))
    e2e = E2E_LEGS * max(1, args.steps) + 1  # + the untimed period before the legs
    return max(cfg.get("t_max", 0), cfg.get("pre_periods", 0) + args.warmup + args.steps + prof + e2e)


# --------------------------------------------------------- reference arm

def reference_step_fn(ref, corpus, cfg, sub_docs: int, n_threads: int, t_max: int, seed: int = 1):
    """One reference period (sampler.cpp:307-333) on a bounded sub-batch, through the
    compiled reference's own sddmm / sample_counts / update_model with n_threads."""
    from oracle import CorpusArrays
    K, W = cfg["n_topics"], corpus.n_words
    rng = np.random.default_rng(seed)
    phi = 1.0 + 0.1 * rng.random((K, W))
    phi /= phi.sum(1, keepdims=True)
    batch_size = max(1, int(round(cfg["batch_fraction"] * corpus.n_docs)))
    state = {"t": 0}

    def step():
        t = state["t"]
        state["t"] += 1
        ids = rng.choice(corpus.n_docs, size=min(sub_docs, batch_size), replace=False)
        sub = CorpusArrays(*_subset(corpus, ids), W)
        local = np.arange(len(ids), dtype=np.int32)
        theta = np.full((len(ids), K), 0.1 + 1.0 / K)
        tb = theta.copy()
        m_t = ref.anneal_m(cfg["schedule"], min(t + 1, t_max), t_max, cfg["m"])
        for sweep in range(cfg["inner_sweeps"]):
            mu = ref.sddmm(tb, phi, sub, local, n_threads)
            tc, pc = ref.sample_counts(tb, phi, mu, sub, local, m_t, seed, t, sweep, n_threads)
            tb = tc / m_t + 0.1
        theta2, phi2 = ref.update_model(theta, phi, local, tc, pc, m_t, ref.rho_schedule(t, 1.0, 0.5),
                                        0.1, 0.01)
        phi[:] = phi2
        tokens = int(sub.counts.astype(np.int64).sum())
        return cfg["inner_sweeps"] * tokens * m_t, int(sub.nnz)

    return step


def _subset(corpus, ids):
    o = corpus.doc_offsets
    lens = o[ids + 1] - o[ids]
    offs = np.zeros(len(ids) + 1, np.int64)
    np.cumsum(lens, out=offs[1:])
    idx = np.concatenate([np.arange(o[d], o[d + 1]) for d in ids])
    return offs, np.ascontiguousarray(corpus.word_ids[idx]), np.ascontiguousarray(
        corpus.counts[idx])


def calibrate_reference(corpus, cfg, n_threads: int, t_max: int):
    """Fit the reference's period time as a + b * docs (a = per-period fixed cost:
    the phi transposes of sddmm/sample_counts, update_model over K x W)."""
    from oracle import Ref
    ref = Ref()
    times = {}
    for n in (64, 512):
        step = reference_step_fn(ref, corpus, cfg, n, n_threads, t_max, seed=7)
        t0 = time.perf_counter()
        step()
        times[n] = time.perf_counter() - t0
    b = max((times[512] - times[64]) / 448.0, 1e-9)
    a = max(times[64] - 64 * b, 0.0)
    return ref, a, b


def reference_sub_batch(corpus, cfg, a, b, budget_s):
    full = max(1, int(round(cfg["batch_fraction"] * corpus.n_docs)))
    if a + b * full <= budget_s:
        return full
    return int(max(64, min(full, (budget_s - a) / b)))


def reference_train_c1(wl: Workload, cfg, n_threads: int):
    """The reference's own train() (sampler.cpp:269-353) on config [0], with eval every 5:
    (samples per run, wall seconds)."""
    from oracle import CorpusArrays, Ref, TrainConfig
    ref = Ref()
    tr = CorpusArrays(wl.train.doc_offsets, wl.train.word_ids, wl.train.counts, wl.train.n_words)
    te = CorpusArrays(wl.heldout.doc_offsets, wl.heldout.word_ids, wl.heldout.counts,
                      wl.heldout.n_words)
    tc = TrainConfig(n_topics=cfg["n_topics"], m=cfg["m"], schedule=cfg["schedule"],
                     batch_fraction=cfg["batch_fraction"], t_max=cfg["t_max"],
                     inner_sweeps=cfg["inner_sweeps"], seed=1, n_threads=n_threads)
    t0 = time.perf_counter()
    _, _, trace = ref.train(tr, tc, te, cfg["eval_every"])
    dt = time.perf_counter() - t0
    samples = cfg["inner_sweeps"] * cfg["m"] * wl.train.n_tokens * cfg["t_max"]  # full batches
    return samples, dt, trace


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    scaling = args.scaling
    record = config_record(cfg, world, scaling)
    if cfg.get("mode") in ("expected", "multinomial") or cfg.get("pre_periods"):
        why = (f"the reference has no {cfg['mode']} mode (sampler.cpp draws Poisson replicas only)"
               if cfg.get("mode") in ("expected", "multinomial") else
               "the converged-model state takes the reference ~100 full periods (~7 min) to reach")
        print(json.dumps({"impl": "reference", "unavailable": why, "config": record}), flush=True)
        return
    n_threads = os.cpu_count() or 1
    wl = Workload(cfg, 1, 0, "strong")  # the whole corpus on the host
    t_max = run_t_max(cfg, args)
    if cfg["corpus"] == "c1":
        samples, dt, _ = reference_train_c1(wl, cfg, n_threads)
        value = samples / dt
        ms = 1000.0 * dt / cfg["t_max"]
        sample_desc = (f"one complete reference train() (oracle/_ref compiled from proj/src): "
                       f"{cfg['t_max']} full-batch periods + eval every {cfg['eval_every']}, "
                       f"{n_threads} threads, {dt:.1f}s")
    else:
        train = wl.train
        ref, a, b = calibrate_reference(train, cfg, n_threads, t_max)
        budget = max(3.0, 180.0 / max(args.steps, 1))
        if os.environ.get("BENCH_REF_BUDGET_S"):  # tests: cap the per-step CPU sample
            budget = float(os.environ["BENCH_REF_BUDGET_S"])
        sub = reference_sub_batch(train, cfg, a, b, budget_s=budget)
        step = reference_step_fn(ref, train, cfg, sub, n_threads, t_max)
        warm = reference_step_fn(ref, train, cfg, 64, n_threads, t_max, seed=3)
        for _ in range(args.warmup):  # CPU code needs no warm-up; keep these cheap
            warm()
        samples = 0.0
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s, _ = step()
            samples += s
        dt = time.perf_counter() - t0
        value = samples / dt
        ms = 1000.0 * dt / args.steps
        sample_desc = (f"reference sddmm+sample_counts x{cfg['inner_sweeps']} + update_model per "
                       f"step on a random {sub}-doc batch (full batch = "
                       f"{int(round(cfg['batch_fraction'] * train.n_docs))} docs; oracle/_ref "
                       f"compiled from proj/src, {n_threads} threads; fitted period time "
                       f"{a:.2f}s + {b * 1e3:.2f}ms/doc)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": record,
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": n_threads,
                         "kind": "reference", "sample": sample_desc},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- our arm

def bytes_per_unit(cfg, final_sweep: bool) -> tuple[int, int]:
    """SURVEY.md 8(d) algorithmic bytes at the element sizes the mode computes in:
    per batch nonzero 8 (word id + count) + e_phi K (phi row) [+ e_cnt K (phi-count row),
    final sweep only: earlier sweeps scatter no phi counts]; per batch doc 8 + e_th K
    (theta row) + e_cnt K (theta counts).  Parity: f64 phi/theta, int32 counts;
    expected: f64 rows and f64 counts; throughput and multinomial: f32 rows, int32 counts."""
    K = cfg["n_topics"]
    mode = cfg.get("mode", "parity")
    e_row, e_cnt = {"expected": (8, 8), "throughput": (4, 4), "multinomial": (4, 4)}.get(mode, (8, 4))
    # which sweeps scatter phi counts: the final one; every one in expected mode and in
    # the parity kernel's multi-slice shapes (K != 256)
    scatter = final_sweep or mode == "expected" or (mode == "parity" and K != 256)
    per_nnz = 8 + e_row * K + (e_cnt * K if scatter else 0)
    per_doc = 8 + e_row * K + e_cnt * K
    return per_nnz, per_doc


def run_ours(args, cfg):
    import torch
    world, rank, local = dist_env()
    # BENCH_SHARE_GPU=1 (testing the multi-rank path on a one-GPU box): every
    # rank on cuda:0 over gloo -- NCCL refuses two ranks on one device; the
    # numbers of such a run are not a measurement
    share = os.environ.get("BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        nccl_v = torch.cuda.nccl.version() if not share else None
        print(f"[bench] rank {rank}/{world} cuda:{local} backend "
              f"{dist.get_backend()} nccl {nccl_v}", file=sys.stderr, flush=True)
    from paper_1409_5402_b200 import distributed as DIST
    from paper_1409_5402_b200 import samelda as S

    scaling = args.scaling
    ctx = S.Context(local)
    # one dedicated (non-blocking) stream for torch and the context: events,
    # collectives and kernels are all ordered on it, and nothing serialises
    # against the legacy default stream
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    wl = Workload(cfg, world, rank, scaling)
    train = wl.train
    t_max = run_t_max(cfg, args)
    scfg = S.SamplerConfig(n_topics=cfg["n_topics"], m=cfg["m"], schedule=cfg["schedule"],
                           batch_fraction=cfg["batch_fraction"], inner_sweeps=cfg["inner_sweeps"],
                           t_max=t_max, seed=1,
                           mode={"expected": S.MODE_EXPECTED, "throughput": S.MODE_THROUGHPUT,
                                 "multinomial": S.MODE_MULTINOMIAL}.get(
                               cfg.get("mode"), S.MODE_PARITY))
    trainer = S.Trainer(train, scfg, ctx=ctx)
    if rank == 0:
        trainer.set_heldout(wl.heldout, seed=1)
    engine = DIST.CudaEngine(trainer, local)
    sharded = DIST.ShardedTrainer(engine, wl.D_global, wl.doc_lo, wl.doc_lo + train.n_docs,
                                  train.doc_tokens(), cfg["batch_fraction"], 1, cfg["m"],
                                  cfg["schedule"], t_max)

    def period(t, result_buf=None):
        assert t == sharded.t
        st = sharded.period()
        # the step's result: batch theta rows, copied D2H into a page-locked
        # host buffer on the trainer stream (no host wait; read back by the
        # barrier that closes the timed region)
        out = trainer.batch_theta_async(st.owned_docs, result_buf) if result_buf is not None else None
        return st.owned_tokens, st.m_t, st.owned_docs, out

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            torch.cuda.synchronize()

    def over_ranks(x: float, op: str) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    # page-locked result buffers of the end-to-end leg, allocated up front; the
    # last warm-up period already reads its result back (copy stream, device
    # row buffers: first-call allocations stay out of every timed region)
    e2e_steps = max(1, args.steps)
    # a rank owns ~batch_fraction x D_global / N docs of each global batch
    # (the call fails loudly if a buffer is ever too small)
    bmax = int(1.25 * cfg["batch_fraction"] * wl.D_global / (world if scaling == "strong" else 1)) + 64
    bmax = min(bmax, train.n_docs)
    bufs = [torch.empty(max(bmax, 1) * cfg["n_topics"], dtype=torch.float64, pin_memory=True).numpy()
            for _ in range(e2e_steps)]
    t = 0
    n_warm = cfg.get("pre_periods", 0) + args.warmup
    for i in range(n_warm):
        period(t, result_buf=bufs[0] if i == n_warm - 1 else None)
        t += 1
    # ---- timed region (device): inputs resident in HBM
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    import gc
    gc.collect()
    gc.disable()  # no collector pauses inside the timed loops
    launches0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    samples = 0.0
    ev0.record(stream)
    for _ in range(args.steps):
        tokens, m_t, _, _ = period(t)
        samples += cfg["inner_sweeps"] * tokens * m_t
        t += 1
    ev1.record(stream)
    barrier()
    dev_ms = over_ranks(ev0.elapsed_time(ev1), "max")
    launches = ctx.launches - launches0
    samples_all = over_ranks(samples, "sum")
    value = samples_all / (dev_ms / 1000.0)

    # ---- per-kernel CUDA-event timing on a separate profiled pass right after
    # the timed region (the profiler synchronises after each sampling launch,
    # so it stays out of the timed region above)
    prof_steps = max(1, min(args.steps, 10))
    trainer.profile(True)
    prof_dev0 = torch.cuda.Event(enable_timing=True)
    prof_dev1 = torch.cuda.Event(enable_timing=True)
    prof_dev0.record(stream)
    for _ in range(prof_steps):
        period(t)
        t += 1
    prof_dev1.record(stream)
    barrier()
    prof = trainer.profile_read()
    trainer.profile(False)
    prof_ms = prof_dev0.elapsed_time(prof_dev1)

    # ---- end to end through the public API with host buffers, right after
    # the profiled pass (the per-period cost drifts up as the model sharpens:
    # more PTRS draws, so the profiled pass comes first and sees the timed
    # region's periods' regime), on as many periods: per step the host batch ids go H2D
    # inside Trainer.period and the batch theta rows (the step's result) come
    # back D2H
    # the clock sampler (nvidia-smi, polling every 25 ms) has covered the timed
    # region and the profiled pass; it stops here, outside every timed region:
    # its polls take driver locks (one-off ~0.1 s stalls of the host-side legs
    # below), and stopping it stalls the next CUDA calls -- absorbed by the
    # pause and one untimed period before the legs
    clk = clocks.stop()
    time.sleep(0.5)
    period(t, result_buf=bufs[0])
    t += 1
    legs = []
    for _ in range(E2E_LEGS):
        barrier()
        h2d = d2h = 0
        samples_e2e = 0.0
        t0 = time.perf_counter()
        for i in range(e2e_steps):
            tokens, m_t, nb, out = period(t, result_buf=bufs[i])
            samples_e2e += cfg["inner_sweeps"] * tokens * m_t
            h2d += nb * 4 + (nb + 1) * 8
            d2h += out.nbytes + 4
            t += 1
        barrier()
        e2e_s = over_ranks(time.perf_counter() - t0, "max")
        legs.append(over_ranks(samples_e2e, "sum") / e2e_s)
    e2e_value = max(legs)
    e2e = {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d // e2e_steps,
           "d2h_bytes_per_step": d2h // e2e_steps,
           "legs": [round(v, 1) for v in legs],
           "how": f"Trainer periods through the C ABI: host batch ids H2D, batch theta rows D2H; "
                  f"best of {E2E_LEGS} legs of {e2e_steps} periods (all in 'legs')"}
    gc.enable()


    # C1: the whole train() through the drop-in entry point (samelda_cu_train),
    # host buffers in and out, eval every 5 -- the call the reference's C++
    # train() shim makes, against the reference's own train()
    if cfg["corpus"] == "c1" and world == 1:
        tcfg = S.SamplerConfig(n_topics=cfg["n_topics"], m=cfg["m"], schedule=cfg["schedule"],
                               batch_fraction=cfg["batch_fraction"],
                               inner_sweeps=cfg["inner_sweeps"], t_max=cfg["t_max"], seed=1)
        runs = []
        for i in range(6):  # the first (untimed) loads the evaluation kernels
            c2 = S.Context(local)  # fresh context: corpus upload, init, everything
            t0 = time.perf_counter()
            _, trace = S.train(train, tcfg, wl.heldout, cfg["eval_every"], ctx=c2)
            if i:
                runs.append(time.perf_counter() - t0)
            c2.close()
        run_s = min(runs)
        s_run = cfg["inner_sweeps"] * cfg["m"] * train.n_tokens * cfg["t_max"]
        corpus_bytes = (train.doc_offsets.nbytes + train.word_ids.nbytes + train.counts.nbytes +
                        wl.heldout.doc_offsets.nbytes + wl.heldout.word_ids.nbytes +
                        wl.heldout.counts.nbytes)
        W, K = train.n_words, cfg["n_topics"]
        e2e = {"value": s_run / run_s, "unit": "samples/s",
               "h2d_bytes_per_step": int((corpus_bytes + 4 * train.n_docs * cfg["t_max"]) / cfg["t_max"]),
               "d2h_bytes_per_step": int(8 * (K * W + train.n_docs * K) / cfg["t_max"]),
               "how": f"samelda_cu_train (drop-in train(), sampler.cpp:269-353): fresh context, "
                      f"{cfg['t_max']} periods, eval every {cfg['eval_every']}, model download; "
                      f"best of 5 runs after an untimed one, {run_s:.3f}s", "final_ll": trace[-1]["ll"]}

    heldout_ll = trainer.evaluate() if rank == 0 else None

    # the drop-in entry point at this shape: samelda_cu_train (what the
    # reference's C++ train() shim calls) from host buffers on a fresh context
    # -- corpus upload, init, 20 periods, one held-out evaluation, model
    # download -- beside the reference arm's period rate
    dropin = None
    if world == 1 and cfg["corpus"] != "c1" and cfg.get("mode", "parity") == "parity":
        T = 20
        tcfg = S.SamplerConfig(n_topics=cfg["n_topics"], m=cfg["m"], schedule=cfg["schedule"],
                               batch_fraction=cfg["batch_fraction"],
                               inner_sweeps=cfg["inner_sweeps"], t_max=T, seed=1)
        runs = []
        for _ in range(3):
            c3 = S.Context(local)
            t0 = time.perf_counter()
            _, dtrace = S.train(train, tcfg, wl.heldout, T, ctx=c3)
            runs.append(time.perf_counter() - t0)
            c3.close()
        d_s = min(runs)
        tokens_run = float(dtrace[-1]["passes"]) * train.n_tokens
        dropin = {"value": cfg["inner_sweeps"] * cfg["m"] * tokens_run / d_s, "unit": "samples/s",
                  "seconds": d_s, "periods": T, "runs_seconds": [round(r, 4) for r in runs],
                  "how": "samelda_cu_train (drop-in train(), sampler.cpp:269-353) on a fresh "
                         "context each run: corpus upload, init, 20 periods, one held-out "
                         "evaluation, model download (phi W x K + theta D x K, f64); best of 3",
                  "final_ll": dtrace[-1]["ll"]}

    # ---- roofline of the dominant kernel (sampling), algorithmic bytes per sweep kind
    peaks, peaks_kind = load_peaks()
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    n_sweeps = cfg["inner_sweeps"]
    nnz_per_launch = prof["nnz"] / max(prof["sample_launches"], 1)
    docs_per_launch = prof["docs"] / max(prof["sample_launches"], 1)
    sweeps = {}
    for kind, final in (("first", False), ("last", True)):
        n = prof[f"sample_{kind}_launches"]
        if n == 0:
            continue
        pn, pd = bytes_per_unit(cfg, final)
        b = nnz_per_launch * pn + docs_per_launch * pd
        ms = prof[f"sample_{kind}_ms"] / n
        sweeps[kind] = {"launches": n, "avg_launch_ms": ms, "alg_bytes_per_launch": b,
                        "achieved_gbs": b / (ms / 1e3) / 1e9 if ms > 0 else 0.0}
    alg_bytes = sum(s["alg_bytes_per_launch"] * s["launches"] for s in sweeps.values())
    sample_ms = prof["sample_ms"]
    achieved = alg_bytes / (sample_ms / 1000.0) / 1e9 if sample_ms > 0 else 0.0
    for s in sweeps.values():
        s["frac"] = s["achieved_gbs"] / peak
    traffic = dram = None
    tfile = os.path.join(ROOT, "profiles", "sample_kernel_traffic.json")
    if os.path.exists(tfile):
        try:
            entry = json.load(open(tfile)).get(args.config, {})
            traffic = entry.get("dram_bytes_per_launch")
            if traffic:
                dram_gbs = traffic / (sample_ms / max(prof["sample_launches"], 1) / 1e3) / 1e9
                dram = {"gbs": dram_gbs, "frac": dram_gbs / peak, "source": entry.get("source")}
        except (OSError, ValueError):
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            n_threads = os.cpu_count() or 1
            if cfg["corpus"] == "c1":
                s_ref, cdt, _ = reference_train_c1(wl, cfg, n_threads)
                cpu = {"value": s_ref / cdt, "unit": "samples/s", "cores": n_threads,
                       "kind": "reference",
                       "sample": f"one complete reference train() ({cfg['t_max']} periods, eval "
                                 f"every {cfg['eval_every']}), oracle/_ref compiled from proj/src, "
                                 f"{n_threads} threads, {cdt:.1f}s"}
            else:
                ref, a, b = calibrate_reference(train, cfg, n_threads, t_max)
                sub = reference_sub_batch(train, cfg, a, b, budget_s=25.0)
                step = reference_step_fn(ref, train, cfg, sub, n_threads, t_max)
                c0 = time.perf_counter()
                s, _ = step()
                cdt = time.perf_counter() - c0
                cpu = {"value": s / cdt, "unit": "samples/s", "cores": n_threads,
                       "kind": "reference",
                       "sample": f"1 reference period (sddmm+sample_counts x{n_sweeps} + "
                                 f"update_model) on a random {sub}-doc batch (full batch "
                                 f"{int(round(cfg['batch_fraction'] * train.n_docs))}), oracle/_ref "
                                 f"compiled from proj/src, {n_threads} threads, {cdt:.1f}s"}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "samples/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    corpus = {"train_docs": wl.D_global, "train_nnz_rank0": train.nnz,
              "train_tokens_rank0": train.n_tokens, "docs_rank0": train.n_docs,
              "heldout_docs": wl.heldout.n_docs if wl.heldout is not None else None,
              "generate_s": round(wl.gen_s, 2)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": {"throughput": "f32", "multinomial": "f32"}.get(cfg.get("mode"), "f64"),
            "data": "synthetic",
            "config": config_record(cfg, world, scaling),
            "corpus": corpus,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "model": "SURVEY 8(d) algorithmic bytes per launch: per batch nonzero "
                                  "8 + 8K (f64 phi row) + 4K (int32 phi-count row, final sweep "
                                  "only), per batch doc 8 + 12K; rows re-read from L2 count, so "
                                  "frac can exceed the DRAM fraction -- see dram",
                         "kernel": {"expected": "k_expected", "throughput": "k_sample_thru",
                                    "multinomial": "k_sample_multi"}.get(
                             cfg.get("mode"), "k_sample_v2 + deferred (parity)"),
                         "peak_kind": peaks_kind, "per_sweep": sweeps, "dram": dram,
                         "alg_bytes_per_launch": alg_bytes / max(prof["sample_launches"], 1),
                         "avg_launch_ms": sample_ms / max(prof["sample_launches"], 1),
                         "sample_share_of_step": sample_ms / prof_ms if prof_ms else None,
                         "mstep_ms_per_step": prof["mstep_ms"] / prof_steps,
                         "deferred_records_per_launch": prof["deferred"] / max(prof["sample_launches"], 1),
                         "profiled_steps": prof_steps},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "dropin_train": dropin,
            "gpu_launches": launches,
            "clocks": clk,
            "heldout_ll": heldout_ll,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="nytimes", choices=sorted(CONFIGS) + sorted(ALIASES))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.config = ALIASES.get(args.config, args.config)
    cfg = CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
