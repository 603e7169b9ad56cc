"""Corpus ingest measurement: the NYTimes-shaped
synthetic corpus written as a UCI docword/vocab pair, loaded by
load_uci_bow -- this build's parallel mmap parser (all host threads) and the
compiled reference's iostream parser (oracle/_ref, on a bounded sample: the
first `--ref-docs` documents) -- plus the binary CSR cache.  Results are
checked equal (same CSR) and printed as one JSON line.

    python tools/ingest_bench.py [--config nytimes] [--ref-docs 30000] [--dir /tmp/ingest]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1409_5402_b200 import samelda as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="nytimes")
ap.add_argument("--ref-docs", type=int, default=30000)
ap.add_argument("--dir", default="/tmp/samelda_ingest")
args = ap.parse_args()
os.makedirs(args.dir, exist_ok=True)
cfg = bench.CONFIGS[args.config]
from paper_1409_5402_b200 import synth  # noqa: E402
full = synth.preset(cfg["corpus"], seed=1)
full.vocab = [f"w{i}" for i in range(full.n_words)]
dw, vb = os.path.join(args.dir, "docword.txt"), os.path.join(args.dir, "vocab.txt")
t0 = time.perf_counter()
S.save_uci_bow(full, dw, vb)
t_save = time.perf_counter() - t0
size = os.path.getsize(dw)

t0 = time.perf_counter()
ours = S.load_uci_bow(dw, vb)
t_load = time.perf_counter() - t0
assert np.array_equal(ours.doc_offsets, full.doc_offsets)
assert np.array_equal(ours.word_ids, full.word_ids) and np.array_equal(ours.counts, full.counts)

cache = os.path.join(args.dir, "corpus.csr")
S.save_corpus_cache(ours, cache)
t0 = time.perf_counter()
cached = S.load_corpus_cache(cache)
t_cache = time.perf_counter() - t0
assert np.array_equal(cached.word_ids, full.word_ids)

# bounded reference sample: the first ref_docs documents as their own file
n = min(args.ref_docs, full.n_docs)
o = full.doc_offsets
sub = S.Corpus(o[:n + 1].copy(), full.word_ids[:o[n]], full.counts[:o[n]], full.n_words,
               full.vocab)
sdw = os.path.join(args.dir, "docword_sample.txt")
S.save_uci_bow(sub, sdw, vb)
ssize = os.path.getsize(sdw)
line = {"workload": cfg["workload"], "docword_bytes": size, "nnz": int(full.nnz),
        "ours": {"load_s": t_load, "MB_per_s": size / t_load / 1e6, "threads": os.cpu_count(),
                 "save_uci_s": t_save, "cache_load_s": t_cache,
                 "cache_GB_per_s": os.path.getsize(cache) / t_cache / 1e9}}
from oracle import Ref, have_ref  # noqa: E402  (test infrastructure: the reference's CPU loader)
if have_ref():
    ref = Ref()
    t0 = time.perf_counter()
    r = ref.load_uci_bow(sdw, vb)
    t_ref = time.perf_counter() - t0
    t0 = time.perf_counter()
    ours_s = S.load_uci_bow(sdw, vb)
    t_ours_s = time.perf_counter() - t0
    assert np.array_equal(r[0], ours_s.doc_offsets) and np.array_equal(r[1], ours_s.word_ids)
    line["reference"] = {"sample_docs": n, "sample_bytes": ssize, "load_s": t_ref,
                         "MB_per_s": ssize / t_ref / 1e6, "threads": 1,
                         "ours_same_sample_s": t_ours_s}
    line["speedup_same_sample"] = t_ref / t_ours_s
print(json.dumps(line), flush=True)
