"""CPU tests of the timing model (paper Eqs. 2-7, reference timing.py).

Hand values follow the reference's own tests (pkg/tests/test_timing.py);
when /root/reference is mounted (build container only) every function is
also compared with the reference on random parameters."""

import os
import sys

import numpy as np
import pytest

from paper_1811_03619_b200 import timing as T
from paper_1811_03619_b200.errors import ConfigError


def stages_of(l_up, l_comp, l_comm, split=0.5, l_b=None):
    f = l_comp * split
    b = l_comp - f
    return T.StageTimes(update=l_up, forward=f, backward=b, first_segment_backward=b if l_b is None else l_b,
                        comm=l_comm)


def test_hand_values():
    assert T.t_sync_total(1, stages_of(1, 2, 3)) == 6
    assert T.t_sync_total(100, stages_of(0.1, 0.9, 0.5)) == pytest.approx(150.0)
    assert T.t_pipe_ideal(100, 4, stages_of(0.1, 0.9, 0.5)) == pytest.approx(37.5)
    assert T.t_pipe_limited(10, stages_of(2, 3, 3)) == 50
    assert T.t_pipe_limited(10, stages_of(1, 1, 7)) == 70
    c = T.ClusterParams(workers=4, latency_s=1e-3, byte_time_s=1e-8, reduce_time_s=1e-9, sync_time_s=2e-3,
                        model_bytes=1e6)
    want = 2 * 3 * 1e-3 + 2 * 0.75 * 1e6 * 1e-8 + 0.75 * 1e6 * 1e-9 + 2e-3
    assert T.ring_comm_time(c) == pytest.approx(want)
    assert T.ring_comm_time(T.ClusterParams(workers=1, sync_time_s=0.5)) == 0.5
    assert T.scaling_efficiency(stages_of(1, 1, 1)) == 1.0
    assert T.scaling_efficiency(stages_of(1, 1, 4)) == 0.5


def test_validation():
    with pytest.raises(ConfigError):
        T.StageTimes(backward=1.0, first_segment_backward=2.0)
    with pytest.raises(ConfigError):
        T.ClusterParams(workers=0)
    with pytest.raises(ConfigError):
        T.ClusterParams(workers=2, segments=0)
    with pytest.raises(ConfigError):
        T.scaling_efficiency(T.StageTimes())


def test_recommendation_depth_two_always():
    r = T.recommend_config(stages_of(0.1, 1.0, 5.0), T.ClusterParams(workers=4, latency_s=1.0, model_bytes=1))
    assert r.depth == 2 and r.bound == T.COMM_BOUND and r.comm_mode == T.SEQUENTIAL


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted (GPU box)")
def test_matches_reference_on_random_parameters():
    sys.path.insert(0, REF)
    try:
        from gradpipe import timing as R
    finally:
        sys.path.remove(REF)
    g = np.random.default_rng(0)
    for _ in range(500):
        kw = dict(workers=int(g.integers(1, 12)), latency_s=float(g.uniform(0, 0.01)),
                  byte_time_s=float(g.uniform(0, 1e-7)), reduce_time_s=float(g.uniform(0, 1e-8)),
                  sync_time_s=float(g.uniform(0, 0.01)), model_bytes=float(g.uniform(0, 1e8)),
                  segments=int(g.integers(1, 20)))
        up, comp, comm = (float(v) for v in g.uniform(0, 1, 3))
        split = float(g.uniform(0.1, 0.9))
        fb = float(g.uniform(0, 1)) * comp * (1 - split)
        s = dict(update=up, forward=comp * split, backward=comp * (1 - split), first_segment_backward=fb, comm=comm)
        ours_c, ref_c = T.ClusterParams(**kw), R.ClusterParams(**kw)
        ours_s, ref_s = T.StageTimes(**s), R.StageTimes(**s)
        it = int(g.integers(1, 1000))
        assert T.ring_comm_time(ours_c) == pytest.approx(R.ring_comm_time(ref_c), rel=1e-12)
        assert T.segmented_comm_time(ours_c) == pytest.approx(R.segmented_comm_time(ref_c), rel=1e-12)
        assert T.star_comm_time(ours_c) == pytest.approx(R.star_comm_time(ref_c), rel=1e-12)
        assert T.t_sync_total(it, ours_s) == pytest.approx(R.t_sync_total(it, ref_s), rel=1e-12)
        assert T.t_pipe_ideal(it, 2, ours_s) == pytest.approx(R.t_pipe_ideal(it, 2, ref_s), rel=1e-12)
        assert T.t_pipe_limited(it, ours_s) == pytest.approx(R.t_pipe_limited(it, ref_s), rel=1e-12)
        assert T.t_pipe_seq(it, ours_s, ours_c) == pytest.approx(R.t_pipe_seq(it, ref_s, ref_c), rel=1e-12)
        assert T.t_pipe_segmented(it, ours_s, ours_c) == pytest.approx(R.t_pipe_segmented(it, ref_s, ref_c),
                                                                         rel=1e-12)
        if ours_s.busy > 0:
            assert T.scaling_efficiency(ours_s) == pytest.approx(R.scaling_efficiency(ref_s), rel=1e-12)
        a, b = T.recommend_config(ours_s, ours_c), R.recommend_config(ref_s, ref_c)
        assert (a.depth, a.comm_mode, a.bound) == (b.depth, b.comm_mode, b.bound)


def test_compare_ring_eq5_terms_and_quant8_extension():
    """timing.compare_ring: Eq. 5's four terms (timing.py:119-132) for the
    codec's payload bytes, the 25 % flag of compare_prediction
    (harness.py:687-720), and the quant8-only extension terms."""
    from paper_1811_03619_b200 import timing as T
    p, n = 4, 1_000_000
    a, b, g, S, d = 2e-6, 1 / 700e9, 1 / 400e9, 5e-6, 1e-11
    for codec, w in (("none", 4), ("trunc16", 2), ("quant8", 1)):
        nb = n * w
        eq5 = 2 * (p - 1) * a + 2 * (p - 1) / p * nb * b + (p - 1) / p * nb * g + S
        row = T.compare_ring(eq5, p, codec, n, a, b, g, S, d)
        assert abs(row["eq5_ms"] - eq5 * 1e3) < 1e-12 and not row["flagged"]
        ext = eq5 + ((nb / p * g + (p - 1) / p * n * d) if codec == "quant8" else 0.0)
        assert abs(row["eq5_ext_ms"] - ext * 1e3) < 1e-12
        assert T.compare_ring(eq5 * 1.3, p, codec, n, a, b, g, S, d)["flagged"]


def test_ring_fixed_overhead_is_eq5_residual_on_the_smallest_call():
    """timing.ring_fixed_overhead: measured smallest call minus its Eq. 5
    prediction (never negative); compare_ring's eq5_ext adds it to every
    codec's prediction, the paper's Eq. 5 column is unchanged."""
    from paper_1811_03619_b200 import timing as T
    p, a, b, g, S = 4, 2e-6, 1 / 700e9, 1 / 400e9, 5e-6
    small = 64
    eq5_small = 2 * (p - 1) * a + 2 * (p - 1) / p * 4 * small * b + (p - 1) / p * 4 * small * g + S
    fixed = T.ring_fixed_overhead(eq5_small + 7e-6, p, small, a, b, g, S)
    assert fixed == pytest.approx(7e-6, rel=1e-9)
    assert T.ring_fixed_overhead(eq5_small / 2, p, small, a, b, g, S) == 0.0
    row0 = T.compare_ring(30e-6, p, "trunc16", 650_000, a, b, g, S)
    row = T.compare_ring(30e-6, p, "trunc16", 650_000, a, b, g, S, fixed_s=fixed)
    assert row["eq5_ms"] == row0["eq5_ms"]
    assert row["eq5_ext_ms"] == pytest.approx(row0["eq5_ext_ms"] + 7e-3, rel=1e-9)
    assert row["terms_us"]["ext_fixed_per_call"] == pytest.approx(7.0)


def test_fenced_phases_follow_the_launch_plan():
    """timing.ring_fenced_phases: LL calls publish without releases; the flag
    protocol ends p phases in a release (p - 1 hops + the allgather), codec
    none's direct reduce-scatter 2; compare_ring adds phases x phi to eq5_ext
    only."""
    from paper_1811_03619_b200 import timing as T
    assert T.ring_fenced_phases(4099, 4, 592, "none") == 0           # LL
    assert T.ring_fenced_phases(16_777_216, 2, 592, "none") == 2     # flag, ring
    assert T.ring_fenced_phases(16_777_216, 4, 592, "trunc16") == 4  # flag, ring
    assert T.ring_fenced_phases(16_777_216, 4, 592, "none") == 2     # flag, direct reduce-scatter
    assert T.ring_fenced_phases(100, 1, 592, "none") == 0
    a, b, g, S = 2e-6, 1 / 700e9, 1 / 400e9, 5e-6
    r0 = T.compare_ring(1e-4, 4, "trunc16", 16_777_216, a, b, g, S)
    r1 = T.compare_ring(1e-4, 4, "trunc16", 16_777_216, a, b, g, S, fence_s=6e-6, fenced_phases=4)
    assert r1["eq5_ms"] == r0["eq5_ms"]
    assert r1["eq5_ext_ms"] == pytest.approx(r0["eq5_ext_ms"] + 0.024, rel=1e-9)
    assert r1["terms_us"]["ext_fence_drain"] == pytest.approx(24.0)
