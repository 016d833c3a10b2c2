"""GPU parity of the fused compressed ring AllReduce (csrc/ring.cu).

* emulated ring (all p ranks in one cooperative launch on cuda:0) against
  every golden case the real reference produced (p = 2, 3, 4, 8; 7 sizes;
  4 magnitude variants; 3 codecs) and against the oracle at larger sizes;
* the per-rank ring (one communicator and one cudaLaunchKernel per rank,
  flag / LL protocols, graph replay, sequence wrap): one GPU per rank over
  NVLink P2P when the box has them, else ranks sharing GPUs (same kernel,
  same launch path, peer pointers in local HBM), same checks;
* reference accounting (messages / payload / frame bytes) and error paths.
Bar: bit-exact outputs on every rank (tests the reference's fold order).
"""

import os

import numpy as np
import pytest
import torch

from helpers import assert_bits_equal, real_transport, run_ranks
from oracle import ring as OR

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.fixture(scope="module")
def P():
    import paper_1811_03619_b200 as P
    return P


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "ring_golden.npz"))


def golden_cases(gold, p):
    for k in gold["keys"]:
        k = str(k)
        if k.startswith(f"p{p}_"):
            yield k, int(k.split("_c")[1]), list(gold[k.rsplit("_c", 1)[0] + "_in"])


def check_against_golden(P, tr, gold, p):
    for k, codec, ins in golden_cases(gold, p):
        def op(r, ep):
            ep.reset_stats()
            y = P.ring_allreduce(ins[r], r, p, ep, P.Codec(codec), iteration=3)
            s = ep.stats
            return y, (s.messages, s.payload_bytes, s.frame_bytes)

        res = run_ranks(tr, op)
        for r, (y, st) in enumerate(res):
            assert_bits_equal(y, gold[k + "_out"], f"{k} rank {r}")
        assert np.array_equal(np.array([st for _, st in res]), gold[k + "_stats"]), k


@pytest.mark.parametrize("p", [2, 3, 4, 8])
def test_emulated_ring_matches_reference_golden(P, gold, p):
    tr = P.EmulatedTransport(p, timeout_s=30.0, max_elems=1 << 14)
    try:
        check_against_golden(P, tr, gold, p)
    finally:
        tr.close()


@pytest.mark.parametrize("p,n", [(2, (1 << 20) + 3), (4, (1 << 21) + 5), (8, 3_000_017), (3, 999_999)])
def test_emulated_ring_large_vs_oracle(P, p, n):
    g = np.random.default_rng((p, n))
    ins = [(g.normal(0, 1, n) * 10.0 ** g.integers(-3, 3)).astype(np.float32) for _ in range(p)]
    tr = P.EmulatedTransport(p, timeout_s=60.0, max_elems=n)
    try:
        for codec in P.Codec:
            want = OR.ring_allreduce_all(ins, int(codec)).outputs[0]
            xs = [torch.from_numpy(v).cuda() for v in ins]
            res = run_ranks(tr, lambda r, ep: P.ring_allreduce(xs[r], r, p, ep, codec, iteration=7))
            for r, y in enumerate(res):
                assert y.is_cuda
                assert_bits_equal(y.cpu().numpy(), want, f"p={p} n={n} {codec.name} rank {r}")
    finally:
        tr.close()


def test_emulated_repeated_calls_reuse_inboxes(P):
    p, n = 4, 50_000
    tr = P.EmulatedTransport(p, timeout_s=30.0, max_elems=n)
    g = np.random.default_rng(11)
    try:
        for it in range(25):
            codec = P.Codec(it % 3)
            m = int(g.integers(1, n))
            ins = [g.normal(0, 1, m).astype(np.float32) for _ in range(p)]
            want = OR.ring_allreduce_all(ins, int(codec)).outputs[0]
            res = run_ranks(tr, lambda r, ep: P.ring_allreduce(ins[r], r, p, ep, codec, iteration=it))
            for y in res:
                assert_bits_equal(y, want, f"iter {it} {codec.name} n={m}")
    finally:
        tr.close()


def test_emulated_nonfinite_raises_codec_error(P):
    p = 4
    tr = P.EmulatedTransport(p, timeout_s=10.0, max_elems=4096)
    ins = [np.ones(1000, np.float32) for _ in range(p)]
    ins[2][500] = np.nan
    try:
        with pytest.raises(P.CodecError):
            run_ranks(tr, lambda r, ep: P.ring_allreduce(ins[r], r, p, ep, P.Codec.TRUNC16))
        # the transport stays usable after a codec error
        ins[2][500] = 1.0
        res = run_ranks(tr, lambda r, ep: P.ring_allreduce(ins[r], r, p, ep, P.Codec.TRUNC16))
        assert np.all(res[0] == 4.0)
    finally:
        tr.close()


def test_single_rank_is_identity(P):
    tr = P.EmulatedTransport(1, max_elems=16)
    vec = np.array([5.0, -1.0], np.float32)
    out = P.ring_allreduce(vec, 0, 1, tr.endpoint(0), P.Codec.QUANT8)
    assert np.array_equal(out, vec)
    tr.close()


def test_rank_mismatch_rejected(P):
    tr = P.EmulatedTransport(2, max_elems=16)
    with pytest.raises(P.CollectiveError):
        P.ring_allreduce(np.ones(4, np.float32), 1, 2, tr.endpoint(0))
    tr.close()


# ------------------------------------- per-rank launches (real multi-GPU path)

# one GPU per rank over NVLink when the box has them, else ranks share GPUs
multigpu = pytest.mark.skipif(NGPU < 1, reason="needs a GPU")


@multigpu
@pytest.mark.parametrize("p", [4, 8])
def test_p2p_ring_matches_reference_golden(P, gold, p):
    """Per-rank launches; p = 8 pairs ranks on 4 GPUs (or shares one)."""
    tr = real_transport(P, p, timeout_s=30.0, max_elems=1 << 14)
    try:
        check_against_golden(P, tr, gold, p)
    finally:
        tr.close()


@multigpu
@pytest.mark.parametrize("n", [1, 4099, (1 << 22) + 3, 25_557_032])
def test_p2p_ring_large_vs_oracle(P, n):
    p = 4
    g = np.random.default_rng(n)
    ins = [g.normal(0, 1, n).astype(np.float32) for _ in range(p)]
    tr = real_transport(P, p, timeout_s=60.0, max_elems=n)
    try:
        for codec in P.Codec:
            want = OR.ring_allreduce_all(ins, int(codec)).outputs[0]
            xs = [torch.from_numpy(v).to(tr.endpoint(r).device) for r, v in enumerate(ins)]
            res = run_ranks(tr, lambda r, ep: P.ring_allreduce(xs[r], r, p, ep, codec, iteration=1))
            for r, y in enumerate(res):
                assert y.device == tr.endpoint(r).device
                assert_bits_equal(y.cpu().numpy(), want, f"n={n} {codec.name} rank {r}")
    finally:
        tr.close()


@multigpu
def test_p2p_timeout_produces_diagnostic(P):
    tr = real_transport(P, 2, timeout_s=0.5, max_elems=64)
    try:
        with pytest.raises(P.CollectiveError, match="reduce-scatter step 0"):
            P.ring_allreduce(np.ones(8, np.float32), 0, 2, tr.endpoint(0))
    finally:
        tr.close()


@multigpu
def test_p2p_failure_poisons_every_later_call(P):
    """After one rank timed out, the abort stays on every rank: a later call
    on the healthy rank ends at once as a consequence of the peer's failure
    instead of waiting out its own timeout (the reference's run ends at the
    first failed recv, collective.py:157-161)."""
    import time
    tr = real_transport(P, 2, timeout_s=1.0, max_elems=1 << 12)
    try:
        with pytest.raises(P.CollectiveError, match="timed out"):
            P.ring_allreduce(np.ones(8, np.float32), 0, 2, tr.endpoint(0))
        t0 = time.perf_counter()
        with pytest.raises(P.CollectiveError, match="aborted after a peer failed"):
            P.ring_allreduce(np.ones(8, np.float32), 1, 2, tr.endpoint(1))
        assert time.perf_counter() - t0 < 0.5
    finally:
        tr.close()


@multigpu
@pytest.mark.parametrize("n,ll", [(300_007, 0), (50_001, None)])  # flag protocol / LL protocol
def test_p2p_ring_in_cuda_graph_replays_bit_exact(P, n, ll):
    """The call sequence number lives on the device, so one captured launch
    can be replayed as many calls (what graph-captured training steps need)."""
    from paper_1811_03619_b200.collective import allreduce_into
    from paper_1811_03619_b200.engine import capture
    p = 2
    g = np.random.default_rng(5)
    ins = [g.normal(0, 1, n).astype(np.float32) for _ in range(p)]
    want = {c: OR.ring_allreduce_all(ins, int(c)).outputs[0] for c in P.Codec}
    tr = real_transport(P, p, timeout_s=30.0, max_elems=n, ll_max_bytes=ll)

    def op(r, ep):
        dev = ep.device
        with torch.cuda.device(dev):
            x = torch.from_numpy(ins[r]).to(dev)
            outs = {c: torch.empty_like(x) for c in P.Codec}
            s = torch.cuda.Stream(dev)
            graph = torch.cuda.CUDAGraph()
            with capture(graph, s):  # no device-wide sync: the other rank may share this GPU
                for c in P.Codec:
                    allreduce_into(x, outs[c], ep, c, 1, s)
            got = []
            for _ in range(4):
                with torch.cuda.stream(s):  # the rank's own stream (ranks may share a GPU)
                    for o in outs.values():
                        o.zero_()
                    graph.replay()
                s.synchronize()
                got.append({c: o.cpu().numpy() for c, o in outs.items()})
            ep._check_errors(n)
            return got

    try:
        res = run_ranks(tr, op)
        for r in range(p):
            for rep in res[r]:
                for c in P.Codec:
                    assert_bits_equal(rep[c], want[c], f"rank {r} {c.name}")
    finally:
        tr.close()


@multigpu
@pytest.mark.parametrize("n,ll", [(8, None), (300_007, 0)])  # LL protocol / flag protocol
def test_p2p_iteration_tag_mismatch_is_a_header_error(P, n, ll):
    """collective.py:52-64: a block carrying another iteration tag is rejected
    (both wire protocols validate the slot header with chunk 0)."""
    tr = real_transport(P, 2, timeout_s=5.0, max_elems=n, ll_max_bytes=ll)
    try:
        xs = [torch.ones(n, device=tr.endpoint(r).device) for r in range(2)]
        with pytest.raises(P.CollectiveError, match="iteration tag"):
            run_ranks(tr, lambda r, ep: P.ring_allreduce(xs[r], r, 2, ep, P.Codec.TRUNC16, iteration=1 + r))
    finally:
        tr.close()


@multigpu
def test_p2p_ll_threshold_and_protocol_switching(P):
    """Sizes either side of the LL threshold (at p = 2, blocks whose payload
    incl. 16 elements of slack is <= 2 MiB use the sequence-tagged LL slots,
    larger ones the flag protocol), called alternately on one communicator:
    every result equals the reference's, so neither protocol ever reads the
    other's stale bytes."""
    p = 2
    t = 2 * ((2 << 20) // 4 - 16)  # fp32 threshold; trunc16's is twice that, quant8's 4x
    sizes = [8, t - 1, t, t + 1, t + 33, 2 * t, 2 * t + 2, 4 * t + 2, 1_000_003, 8, t, 5]
    tr = real_transport(P, p, timeout_s=30.0, max_elems=max(sizes))
    try:
        for k, n in enumerate(sizes):
            g = np.random.default_rng(k)
            ins = [g.normal(0, 1, n).astype(np.float32) for _ in range(p)]
            for codec in P.Codec:
                want = OR.ring_allreduce_all(ins, int(codec)).outputs[0]
                xs = [torch.from_numpy(v).to(tr.endpoint(r).device) for r, v in enumerate(ins)]
                res = run_ranks(tr, lambda r, ep: P.ring_allreduce(xs[r], r, p, ep, codec, iteration=k))
                for r, y in enumerate(res):
                    assert_bits_equal(y.cpu().numpy(), want, f"n={n} {codec.name} rank {r}")
    finally:
        tr.close()


@multigpu
def test_p2p_ring_across_call_sequence_wrap(P):
    """Sequence numbers cycle 1 .. 2^32-1 and every check is an equality:
    calls straddling the wrap (both wire protocols, every codec, fused
    variants included via the graph test's allreduce_into path) stay exact."""
    from paper_1811_03619_b200 import _lib
    p = 2
    tr = real_transport(P, p, timeout_s=30.0, max_elems=300_007, ll_max_bytes=256 << 10)
    try:
        for r in range(p):
            _lib.call("gp_comm_set_call_counter", tr.endpoint(r)._comm, 0xFFFFFFFF - 4)
        for k in range(4):
            for n in (1000, 300_007):  # LL / flag protocol
                g = np.random.default_rng(100 * k + n % 7)
                ins = [g.normal(0, 1, n).astype(np.float32) for _ in range(p)]
                for codec in P.Codec:
                    want = OR.ring_allreduce_all(ins, int(codec)).outputs[0]
                    xs = [torch.from_numpy(v).to(tr.endpoint(r).device) for r, v in enumerate(ins)]
                    res = run_ranks(tr, lambda r, ep: P.ring_allreduce(xs[r], r, p, ep, codec, iteration=k))
                    for r, y in enumerate(res):
                        assert_bits_equal(y.cpu().numpy(), want, f"k={k} n={n} {codec.name} rank {r}")
    finally:
        tr.close()


@pytest.mark.parametrize("p", [3, 2])
def test_empty_vector_ring_matches_reference(P, p):
    """n = 0 (the reference returns empty arrays and still counts 2(p-1)
    messages of 0 payload / 20 frame bytes each; checked against the oracle,
    which reproduces the reference's stats)."""
    emulated = p == 3
    tr = P.EmulatedTransport(p, timeout_s=30.0, max_elems=64) if emulated else real_transport(P, p, timeout_s=30.0,
                                                                                             max_elems=64)
    try:
        ins = [np.zeros(0, np.float32) for _ in range(p)]
        for codec in P.Codec:
            want = OR.ring_allreduce_all(ins, int(codec))

            def op(r, ep):
                ep.reset_stats()
                y = P.ring_allreduce(ins[r], r, p, ep, codec, iteration=2)
                s = ep.stats
                return y, (s.messages, s.payload_bytes, s.frame_bytes)

            res = run_ranks(tr, op)
            for r, (y, st) in enumerate(res):
                assert y.shape == (0,) and y.dtype == np.float32
                w = want.stats[r]
                assert st == (w.messages, w.payload_bytes, w.frame_bytes), (codec, r, st)
    finally:
        tr.close()


def test_call_over_capacity_is_a_config_error(P):
    """A vector longer than the communicator was created for is a caller
    error (ConfigError), reported before any launch."""
    tr = P.EmulatedTransport(2, timeout_s=10.0, max_elems=1000)
    try:
        ins = [np.ones(1001, np.float32) for _ in range(2)]
        with pytest.raises(P.ConfigError, match="capacity"):
            run_ranks(tr, lambda r, ep: P.ring_allreduce(ins[r], r, 2, ep, P.Codec.NONE))
    finally:
        tr.close()


@multigpu
@pytest.mark.parametrize("n,ll", [(300_007, 0), (50_001, None)])  # flag protocol / LL protocol
def test_graph_replayed_ring_checks_the_device_iteration_tag(P, n, ll):
    """A ring captured once in a CUDA graph reads its iteration tag from
    device memory (gp_comm_set_iteration_source), so the reference's _expect
    check (collective.py:52-64) stays live under replay: equal tags replay
    bit-exact, a rank one step ahead is a header error."""
    from paper_1811_03619_b200 import _lib
    from paper_1811_03619_b200.collective import allreduce_into
    from paper_1811_03619_b200.engine import capture
    p = 2
    g = np.random.default_rng(11)
    ins = [g.normal(0, 1, n).astype(np.float32) for _ in range(p)]
    want = OR.ring_allreduce_all(ins, int(P.Codec.TRUNC16)).outputs[0]
    tr = real_transport(P, p, timeout_s=5.0, max_elems=n, ll_max_bytes=ll)
    tags = [[7, 7], [8, 8], [9, 10]]  # the third replay: rank 1 is one iteration ahead

    def op(r, ep):
        dev = ep.device
        with torch.cuda.device(dev):
            x = torch.from_numpy(ins[r]).to(dev)
            out = torch.empty_like(x)
            tag = torch.zeros(1, dtype=torch.int32, device=dev)
            s = torch.cuda.Stream(dev)
            _lib.call("gp_comm_set_iteration_source", ep._comm, tag.data_ptr())
            graph = torch.cuda.CUDAGraph()
            with capture(graph, s):
                allreduce_into(x, out, ep, P.Codec.TRUNC16, 0, s)
            _lib.call("gp_comm_set_iteration_source", ep._comm, None)
            got = []
            for k in range(len(tags)):
                with torch.cuda.stream(s):
                    tag.fill_(tags[k][r])
                    out.zero_()
                    graph.replay()
                s.synchronize()
                try:
                    ep._check_errors(n)
                except P.CollectiveError as e:
                    got.append(str(e))
                    break
                got.append(out.cpu().numpy())
            return got

    try:
        res = run_ranks(tr, op)
    finally:
        tr.close()
    for r in range(p):
        assert len(res[r]) == 3, res[r]
        for k in range(2):
            assert_bits_equal(res[r][k], want, f"rank {r} replay {k}")
    assert any(isinstance(x, str) and "iteration tag" in x for x in (res[0][2], res[1][2])), (res[0][2], res[1][2])
