"""Multi-GPU inside the C ABI (samelda_cu_group_*, csrc/group.cu): one process,
documents sharded over the group's devices, the per-period W x K count exchange,
the replicated M-step.  The sharded train() must equal the single-context
train() (samelda_cu_train) bit for bit -- phi, every theta row, the ll trace --
in the integer-count modes, for any number of members.  On this one-GPU box:
a one-member group over NCCL (ncclCommInitAll on one device: the library loads,
the communicator forms, the all-reduce runs in place) and groups repeating
device 0 (the device-side exchange); on a box with >= 2 GPUs, NCCL over
distinct devices."""
from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

K, SEED = 16, 5


@pytest.fixture(scope="module")
def data():
    from oracle import Port
    from paper_1409_5402_b200 import samelda as S
    port = Port()
    g = port.make_corpus(150, 80, 5, 30.0, 12)
    tr, te = port.split_holdout(g, 0.2, 3)
    return S, S.Corpus.of(tr), S.Corpus.of(te)


def _same(S, data_, devices, mode, schedule="linear", bf=0.3):
    S_, tr, te = data_
    cfg = S.SamplerConfig(n_topics=K, m=25.0, schedule=schedule, t_max=6, batch_fraction=bf,
                          seed=SEED, mode=mode)
    want, wtrace = S.train(tr, cfg, te, 2, ctx=S.Context(0))
    g = S.Group(devices)
    got, gtrace = g.train(tr, cfg, te, 2)
    np.testing.assert_array_equal(got.phi, want.phi)
    np.testing.assert_array_equal(got.theta, want.theta)
    assert [r["ll"] for r in gtrace] == [r["ll"] for r in wtrace]
    assert [r["m_t"] for r in gtrace] == [r["m_t"] for r in wtrace]
    return g


@pytest.mark.parametrize("mode", [0, 2], ids=["parity", "throughput"])
def test_one_member_group_over_nccl(data, mode):
    S = data[0]
    g = _same(S, data, [0], mode)
    assert g.uses_nccl


@pytest.mark.parametrize("n", [2, 3, 7])
@pytest.mark.parametrize("mode", [0, 2], ids=["parity", "throughput"])
def test_repeated_device_groups_equal_one_gpu(data, n, mode):
    S = data[0]
    g = _same(S, data, [0] * n, mode, schedule="constant" if n == 3 else "linear")
    assert not g.uses_nccl


def test_more_members_than_batch_documents(data):
    """bf small: most members own no document of a batch (empty owned batches)."""
    S = data[0]
    _same(S, data, [0] * 5, 0, bf=0.02)


def test_expected_mode_group_close(data):
    """Expected counts are f64 sums: the exchange's order may differ from one GPU's
    (tolerance 1e-12 relative, not bit-identity)."""
    S, tr, te = data
    cfg = S.SamplerConfig(n_topics=K, m=25.0, t_max=4, batch_fraction=0.3, seed=SEED, mode=1)
    want, _ = S.train(tr, cfg, ctx=S.Context(0))
    got, _ = S.Group([0, 0]).train(tr, cfg)
    np.testing.assert_allclose(got.phi, want.phi, rtol=1e-12, atol=0)


def test_mixed_device_list_rejected():
    from paper_1409_5402_b200 import samelda as S
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 devices to form a mixed list")
    with pytest.raises(S.ConfigError):
        S.Group([0, 0, 1])


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode", [0, 2], ids=["parity", "throughput"])
def test_nccl_group_over_distinct_devices(data, mode):
    S = data[0]
    n = torch.cuda.device_count()
    g = _same(S, data, list(range(n)), mode)
    assert g.uses_nccl
