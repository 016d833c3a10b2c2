"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py). CPU only; no GPU, no /root/reference needed."""

import os

import numpy as np
import pytest

from oracle import codec as C
from oracle import engine as E
from oracle import ring as R

from golden.cases import ENGINE_CASES

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def codec_gold():
    return np.load(os.path.join(GOLD, "codec_golden.npz"))


@pytest.fixture(scope="module")
def ring_gold():
    return np.load(os.path.join(GOLD, "ring_golden.npz"))


@pytest.fixture(scope="module")
def engine_gold():
    return np.load(os.path.join(GOLD, "engine_golden.npz"))


def test_codec_known_answers():
    # test_compression.py:40-51 and :92-124
    _, pl = C.encode(np.array([1.0], np.float32), C.TRUNC16)
    assert int(pl[0]) == 0x3F80
    _, pl = C.encode(np.array([np.float32(np.pi)], np.float32), C.TRUNC16)
    assert int(pl[0]) == 0x4049
    assert C.decode(C.TRUNC16, 0, pl)[0] == np.float32(3.140625)
    s, pl = C.encode(np.array([0.0, 1.0, -1.0, 0.5], np.float32), C.QUANT8)
    assert list(pl) == [0, 127, -127, 64]
    s, pl = C.encode(np.array([127.0, 2.5, -2.5, 0.5, -0.5], np.float32), C.QUANT8)
    assert s == np.float32(1.0) and list(pl) == [127, 3, -3, 1, -1]
    s, pl = C.encode(np.zeros(33, np.float32), C.QUANT8)
    assert s == 0.0 and not pl.any()
    with pytest.raises(C.OracleCodecError):
        C.encode(np.array([1.0, np.nan], np.float32), C.NONE)


def test_codec_matches_reference_golden(codec_gold):
    for i in range(int(codec_gold["count"][0])):
        x = codec_gold[f"x{i}"]
        _, t16 = C.encode(x, C.TRUNC16)
        assert np.array_equal(t16, codec_gold[f"t16_{i}"]), i
        s, q8 = C.encode(x, C.QUANT8)
        assert np.array_equal(q8, codec_gold[f"q8_{i}"]), i
        assert np.array_equal(np.array([s], np.float32).view(np.uint32),
                              codec_gold[f"q8s_{i}"].view(np.uint32)), i


def test_partition_blocks():
    for n in (0, 1, 7, 16, 4099, 61_100_840):
        for p in (1, 2, 3, 4, 8):
            bl = R.partition_blocks(n, p)
            assert sum(l for _, l in bl) == n
            assert max(l for _, l in bl) - min(l for _, l in bl) <= 1
            assert all(bl[i][0] + bl[i][1] == bl[i + 1][0] for i in range(p - 1))


def test_ring_matches_reference_golden(ring_gold):
    for k in ring_gold["keys"]:
        k = str(k)
        p = int(k.split("_")[0][1:])
        codec = int(k.split("_c")[1])
        ins = list(ring_gold[k.rsplit("_c", 1)[0] + "_in"])
        res = R.ring_allreduce_all(ins, codec, keep_messages=True)
        want = ring_gold[k + "_out"]
        for out in res.outputs:
            assert out.view(np.uint32).tobytes() == want.view(np.uint32).tobytes(), k
        stats = np.array([(s.messages, s.payload_bytes, s.frame_bytes) for s in res.stats])
        assert np.array_equal(stats, ring_gold[k + "_stats"]), k
        log = ring_gold[k + "_log"]
        if p > 1:
            got = np.array([[(m.block, m.wire_bytes) for m in sent] for sent in res.sent])
            assert np.array_equal(got, log), k
        # closed-form fold gives the same bits
        assert R.ring_fold(ins, codec).tobytes() == want.tobytes(), k


def test_ring_schedule_golden_p4_n10(ring_gold):
    # rank 0 sends blocks 0,3,2 | 1,0,3; rank 1 sends 1,0,3 | 2,1,0
    log = ring_gold["p4_n10_v0_c0_log"]
    assert list(log[0][:, 0]) == [0, 3, 2, 1, 0, 3]
    assert list(log[1][:, 0]) == [1, 0, 3, 2, 1, 0]
    assert list(log[0][:, 1]) == [21, 17, 17, 21, 21, 17]


ENGINE_NET = {"log": E.Net("logistic", (8, 3)), "mlp": E.Net("mlp", (8, 16, 12, 3))}


@pytest.mark.parametrize("case", ENGINE_CASES, ids=lambda c: c[0])
def test_engine_trajectory_matches_reference(case, engine_gold):
    name, m, mode, codec, p, T, K, warm, lr, bs, dec = case
    data = E.synthetic_blobs(dim=8, num_classes=3, num_samples=512, seed=1)
    cfg = E.Config(mode=mode, iterations=T, learning_rate=lr, codec=codec, depth=K,
                   batch_size=bs, warmup_epochs=warm, seed=7, lr_decay_every=dec,
                   lr_decay_factor=0.5)
    tr = E.run_trajectory(p, cfg, data, ENGINE_NET[m])
    assert tr.params.tobytes() == engine_gold[name].tobytes(), name
    np.testing.assert_array_equal(np.array(tr.losses[0]), engine_gold[name + "_loss"])
