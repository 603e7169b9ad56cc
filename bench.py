"""SAME factored Gibbs sampler benchmark (BASELINE.json metric and config).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config nytimes|c1|pubmed|k1024]

A step is one SAME period (Algorithm 3; sampler.cpp:307-333) over one
minibatch of the synthetic corpus: inner_sweeps x (SDDMM + Poisson replica
sampling + count scatter) and the M-step.  Metric: sampled token x replica
samples per second = sum over sweeps of (batch tokens x m_t) / time.

Default workload (BASELINE.json configs[1]): NYTimes-shaped synthetic corpus
(300K docs, 102,660 words, ~100M tokens, ~70M nonzeros), K=256, m=100,
batch_fraction 0.05, inner_sweeps 2, parity mode (f64, reference-identical
draws).  N>1 (torchrun): weak scaling -- rank r holds its own NYTimes-shaped
shard of a global corpus of N x 300K docs; one global MinibatchStream, each
rank samples the batch docs it owns, the W x K topic-word counts are
all-reduced over NCCL once per period, the M-step is replicated.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]
    "nytimes": dict(corpus="nytimes", n_topics=256, m=100.0, batch_fraction=0.05,
                    inner_sweeps=2, schedule="constant",
                    workload="NYTimes-shaped synthetic corpus (300K docs, 102,660 vocab, ~100M "
                             "tokens), K=256, m=100, bf=0.05, 2 inner sweeps"),
    # BASELINE.json configs[3] (one GPU holds it; 8xB200 is the published shape)
    "pubmed": dict(corpus="pubmed", n_topics=256, m=100.0, batch_fraction=0.05, inner_sweeps=2,
                   schedule="constant",
                   workload="PubMed-shaped synthetic corpus (8.2M docs, 141,043 vocab, ~730M "
                            "tokens), K=256, m=100, bf=0.05"),
    # the deterministic factored expected-count path (north star (3); z := rate)
    "nytimes-expected": dict(corpus="nytimes", n_topics=256, m=100.0, batch_fraction=0.05,
                             inner_sweeps=2, schedule="constant", mode="expected",
                             workload="NYTimes-shaped synthetic corpus, K=256, m=100, bf=0.05, "
                                      "2 inner sweeps, expected-count mode"),
    # throughput mode: same sampler, own f32 random streams
    # (statistical, not bit, parity with the reference)
    "nytimes-fast": dict(corpus="nytimes", n_topics=256, m=100.0, batch_fraction=0.05,
                         inner_sweeps=2, schedule="constant", mode="throughput",
                         workload="NYTimes-shaped synthetic corpus, K=256, m=100, bf=0.05, "
                                  "2 inner sweeps, throughput mode (f32, own random streams)"),
    # BASELINE.json configs[4]
    "k1024": dict(corpus="nytimes", n_topics=1024, m=50.0, batch_fraction=0.05, inner_sweeps=2,
                  schedule="constant",
                  workload="NYTimes-shaped synthetic corpus, K=1024, m=50, bf=0.05"),
}

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


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


def make_corpus(name: str, shard: int, n_threads: int | None = None):
    from paper_1409_5402_b200 import synth
    return synth.preset(name, seed=1, shard=shard, n_threads=n_threads)


def split_heldout(corpus, frac=0.1):
    """Last `frac` of the (iid) generated docs are held out."""
    from paper_1409_5402_b200.samelda import Corpus
    D = corpus.n_docs
    n_test = max(1, int(round(frac * D)))
    cut = D - n_test
    o = corpus.doc_offsets
    train = Corpus(o[:cut + 1].copy(), corpus.word_ids[:o[cut]], corpus.counts[:o[cut]],
                   corpus.n_words)
    test = Corpus(o[cut:] - o[cut], corpus.word_ids[o[cut]:], corpus.counts[o[cut]:],
                  corpus.n_words)
    return train, test


# --------------------------------------------------------- reference arm

def reference_step_fn(ref, corpus, cfg, sub_docs: int, n_threads: int, seed: int = 1):
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
        m_t = cfg["m"]
        for sweep in range(cfg["inner_sweeps"]):
            mu = ref.sddmm(tb, phi, sub, local, n_threads)
            tc, pc = ref.sample_counts(tb, phi, mu, sub, local, m_t, seed, t, sweep, n_threads)
            tb = tc / m_t + 0.1
        theta2, phi2 = ref.update_model(theta, phi, local, tc, pc, m_t, 0.5, 0.1, 0.01)
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


def calibrate_reference(corpus, cfg, n_threads: int):
    """Fit the reference's period time as a + b * docs (a = per-period fixed cost:
    the phi transposes of sddmm/sample_counts, update_model over K x W)."""
    from oracle import Ref
    ref = Ref()
    times = {}
    for n in (64, 512):
        step = reference_step_fn(ref, corpus, cfg, n, n_threads, seed=7)
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


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    if cfg.get("mode") == "expected":
        print(json.dumps({"impl": "reference",
                          "unavailable": "the reference has no expected-count mode "
                                         "(sampler.cpp draws Poisson replicas only)"}), flush=True)
        return
    n_threads = os.cpu_count() or 1
    corpus = make_corpus(cfg["corpus"], 0)
    train, _ = split_heldout(corpus)
    ref, a, b = calibrate_reference(train, cfg, n_threads)
    budget = max(3.0, 180.0 / max(args.steps, 1))
    if os.environ.get("BENCH_REF_BUDGET_S"):  # tests: cap the per-step CPU sample
        budget = float(os.environ["BENCH_REF_BUDGET_S"])
    sub = reference_sub_batch(train, cfg, a, b, budget_s=budget)
    step = reference_step_fn(ref, train, cfg, sub, n_threads)
    warm = reference_step_fn(ref, train, cfg, 64, n_threads, seed=3)
    for _ in range(args.warmup):  # CPU code needs no warm-up; keep these cheap
        warm()
    samples = 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s, _ = step()
        samples += s
    dt = time.perf_counter() - t0
    value = samples / dt
    line = {
        "impl": "reference", "metric": "sampled tokens/sec (x m replicas)", "value": value,
        "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * dt / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "K": cfg["n_topics"], "m": cfg["m"],
                   "batch_fraction": cfg["batch_fraction"], "inner_sweeps": cfg["inner_sweeps"]},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": n_threads,
                         "kind": "reference",
                         "sample": f"reference sddmm+sample_counts x{cfg['inner_sweeps']} + "
                                   f"update_model per step on a random {sub}-doc batch "
                                   f"(full batch = {int(round(cfg['batch_fraction'] * train.n_docs))}"
                                   f" docs; oracle/_ref compiled from proj/src, {n_threads} "
                                   f"threads; fitted period time {a:.2f}s + {b * 1e3:.2f}ms/doc)"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- our arm

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
    from paper_1409_5402_b200 import samelda as S

    ctx = S.Context(local)
    # one dedicated (non-blocking) stream for torch and the context: events,
    # collectives and kernels are all ordered on it, and nothing serialises
    # against the legacy default stream
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    t_gen = time.perf_counter()
    corpus = make_corpus(cfg["corpus"], rank)
    train, heldout = split_heldout(corpus)
    gen_s = time.perf_counter() - t_gen
    D_local = train.n_docs
    D_global = D_local * world
    doc_base = rank * D_local  # weak scaling: rank r owns global docs [r*D, (r+1)*D)

    scfg = S.SamplerConfig(n_topics=cfg["n_topics"], m=cfg["m"], schedule=cfg["schedule"],
                           batch_fraction=cfg["batch_fraction"], inner_sweeps=cfg["inner_sweeps"],
                           t_max=args.warmup + args.steps + 2 * max(1, min(args.steps, 10)), seed=1,
                           mode={"expected": S.MODE_EXPECTED, "throughput": S.MODE_THROUGHPUT}.get(
                               cfg.get("mode"), S.MODE_PARITY))
    trainer = S.Trainer(train, scfg, ctx=ctx)
    trainer.set_doc_base(doc_base)
    if rank == 0:
        trainer.set_heldout(heldout, seed=1)
    from paper_1409_5402_b200 import distributed as DIST
    engine = DIST.CudaEngine(trainer, local)
    sharded = DIST.ShardedTrainer(engine, D_global, doc_base, doc_base + D_local,
                                  train.doc_tokens(), cfg["batch_fraction"], 1, cfg["m"],
                                  cfg["schedule"], scfg.t_max)

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

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t)
        return float(t.item())

    t = 0
    for _ in range(args.warmup):
        period(t)
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
    dev_ms = max_over_ranks(ev0.elapsed_time(ev1))
    launches = ctx.launches - launches0
    clk = clocks.stop()
    samples_all = sum_over_ranks(samples)
    value = samples_all / (dev_ms / 1000.0)

    # ---- per-kernel CUDA-event timing on a separate profiled pass (the
    # profiler synchronises after each sampling launch, so it stays out of
    # the timed region above)
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

    # ---- end to end through the public API with host buffers: per step the
    # host batch ids go H2D inside Trainer.period and the batch theta rows
    # (the step's result) come back D2H
    e2e_steps = max(1, min(args.steps, 10))
    # a rank owns ~batch_fraction x D_local docs of each global batch (the
    # call fails loudly if a buffer is ever too small)
    bmax = int(1.25 * cfg["batch_fraction"] * D_local) + 64
    bufs = [torch.empty(bmax * cfg["n_topics"], dtype=torch.float64, pin_memory=True).numpy()
            for _ in range(e2e_steps)]
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
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_value = sum_over_ranks(samples_e2e) / e2e_s

    gc.enable()
    heldout_ll = trainer.evaluate() if rank == 0 else None

    # ---- roofline of the dominant kernel (sampling), algorithmic bytes
    K = cfg["n_topics"]
    # SURVEY.md 8(d) per-unit figure at parity-mode element sizes (phi f64
    # "use 8 in place of 4", int32 counts): per batch nonzero 8 (word id +
    # count) + 8K (phi column) + 4K (phi-count column); per batch doc
    # 8 + 8K (theta row) + 4K (theta counts).  This build moves the same
    # 12K + 8 per nonzero (phi32 4K + u64 counts 8K).
    # (expected-count mode: f64 rates -- 8K phi row + 8K f64 RED per nonzero)
    per_nnz = 8 + (16 if cfg.get("mode") == "expected" else 12) * K
    per_doc = 8 + (16 if cfg.get("mode") == "expected" else 12) * K
    alg_bytes = prof["nnz"] * per_nnz + prof["docs"] * per_doc
    sample_ms = prof["sample_ms"]
    peaks, peaks_kind = load_peaks()
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    achieved = alg_bytes / (sample_ms / 1000.0) / 1e9 if sample_ms > 0 else 0.0
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "sample_kernel_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(args.config, {}).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            n_threads = os.cpu_count() or 1
            ref, a, b = calibrate_reference(train, cfg, n_threads)
            sub = reference_sub_batch(train, cfg, a, b, budget_s=25.0)
            step = reference_step_fn(ref, train, cfg, sub, n_threads)
            c0 = time.perf_counter()
            s, _ = step()
            cdt = time.perf_counter() - c0
            cpu = {"value": s / cdt, "unit": "samples/s", "cores": n_threads,
                   "kind": "reference",
                   "sample": f"1 reference period (sddmm+sample_counts x{cfg['inner_sweeps']} + "
                             f"update_model) on a random {sub}-doc batch (full batch "
                             f"{int(round(cfg['batch_fraction'] * train.n_docs))}), oracle/_ref "
                             f"compiled from proj/src, {n_threads} threads, {cdt:.1f}s"}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "samples/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "sampled tokens/sec (x m replicas)", "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "K": K, "m": cfg["m"],
                       "batch_fraction": cfg["batch_fraction"],
                       "inner_sweeps": cfg["inner_sweeps"], "mode": cfg.get("mode", "parity"),
                       "docs_per_gpu": D_local, "nnz_per_gpu": train.nnz,
                       "tokens_per_gpu": train.n_tokens, "parallelism": f"doc-shard x{world}",
                       "l2": "inputs larger than L2 (phi 210 MB f64 + theta 553 MB per GPU; "
                             "random minibatch docs each step)",
                       "corpus_gen_s": round(gen_s, 2)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "model": "SURVEY 8(d) per-nonzero gather bytes (phi row + count row per "
                                  "nonzero, theta rows per doc); rows re-read from L2 are counted, "
                                  "so frac can exceed 1 for an L2-resident kernel -- see traffic "
                                  "for DRAM bytes",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "kernel": {"expected": "k_expected", "throughput": "k_sample_thru"}.get(
                             cfg.get("mode"), "k_sample_v2 + deferred (parity)"), "peak_kind": peaks_kind,
                         "alg_bytes_per_launch": alg_bytes / max(prof["sample_launches"], 1),
                         "avg_launch_ms": sample_ms / max(prof["sample_launches"], 1),
                         "sample_share_of_step": sample_ms / prof_ms if prof_ms else None,
                         "mstep_ms_per_step": prof["mstep_ms"] / prof_steps,
                         "deferred_records_per_launch": prof["deferred"] / max(prof["sample_launches"], 1),
                         "profiled_steps": prof_steps},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "samples/s",
                    "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps},
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
    ap.add_argument("--config", default="nytimes", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
