"""GPU tests of the C-ABI surface around the step loop: setup timing, launch accounting,
record-ring bounds and the zero-allocation read path used by bench.py's e2e leg.  The
spike trains themselves are checked against the oracle in test_gpu_parity.py."""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2102_04681_b200 import build as B
    B.build()
    from paper_2102_04681_b200 import spice
    return spice


def test_setup_times_are_reported(S):
    with S.Network(W.synth(20000, 31, 0.005, seed=3)) as net:
        t = net.setup_times()
        assert 0.0 < t["gen_ms"] <= t["create_ms"]


@pytest.mark.parametrize("kw, per_chunk", [
    ({}, 2),                                     # small network: one k_small + k_advance per 32 steps
    (dict(tile_width=1024), 34),                 # tiled: update, 31 fused, deliver, advance
    (dict(tile_width=1024, unfused=True), 65),   # update + deliver per step, advance
])
def test_launch_accounting(S, kw, per_chunk):
    with S.Network(W.synth(20000, 31, 0.005, seed=3), **kw) as net:
        assert net.launches(32) == per_chunk
        assert net.launches(64) == 2 * per_chunk
        single = net.launches(1)
        assert net.launches(33) == per_chunk + single


def test_record_ring_bounds(S):
    cfg = W.vogels(4000)
    with S.Network(cfg, record_steps=16) as net:
        net.step(40)
        assert len(net.read_spikes(24, 40)) == 16          # the last record_steps steps
        with pytest.raises(S.SpiceError):
            net.read_spikes(20, 40)                         # older than the ring
        with pytest.raises(S.SpiceError):
            net.read_spikes(30, 41)                         # not simulated yet


def test_read_spikes_into_matches_oracle(S):
    """The e2e read path (pinned staging, reused decode buffers) step by step."""
    cfg, T = W.synth(5003, 31, 0.05, seed=21), 64
    o = O.OracleNet(cfg)
    o.step(T)
    want = o.spikes()
    ids = np.zeros(cfg.n, dtype=np.uint32)
    offs = np.zeros(2, dtype=np.uint64)
    with S.Network(cfg, record_steps=8) as net:
        for t in range(T):
            net.step(1)
            k = net.read_spikes_into(t, t + 1, ids, offs)
            assert np.array_equal(ids[:k], want[t]), t
