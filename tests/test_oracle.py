"""CPU: pin the oracle. The C restatement (oracle/pmklc_oracle.c) must agree
with the reference compiled from its own sources (oracle/_ref) and with the
reference's golden vectors."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracles as O

G = Path(__file__).resolve().parent / "golden"


def test_skmer_golden_vectors(port):
    # "CGG" -> 26 (test_skmer.cpp:38-43) and reference outputs on all 36 (s,k)
    for case in json.loads((G / "skmer.json").read_text()):
        tok, res = port.skmer_encode(bytes(case["codes"]), case["s"], case["k"])
        assert tok.tolist() == case["tokens"]
        assert list(res) == case["residual"]


def test_token_count_closed_form(port):
    # test_skmer.cpp:45-58
    for n, s, k, want in [(0, 3, 3, 0), (2, 3, 3, 0), (3, 3, 3, 1), (5, 3, 3, 1), (6, 3, 3, 2),
                          (10, 2, 4, 4), (10, 1, 1, 10)]:
        tok, _ = port.skmer_encode(bytes(n), s, k)
        assert len(tok) == want


def test_quantize_frozen_and_reference_vectors(port):
    # frozen vectors test_coder.cpp:53-70 are the first five cases
    cases = json.loads((G / "quantize.json").read_text())
    assert cases[0]["freqs"] == [63570, 656, 655, 655]
    assert cases[1]["freqs"] == [65533, 1, 1, 1]
    assert cases[3]["freqs"] == [26214, 19661, 13107, 6554]
    assert cases[4]["freqs"] == [21845, 21845, 21846]
    for c in cases:
        p = np.asarray(c["p_bits"], dtype=np.uint32).view(np.float32)
        if c["error"]:
            with pytest.raises(O.CheckerError) as e:
                port.quantize(p)
            assert e.value.errc == c["error"]
        else:
            assert port.quantize(p).tolist() == c["freqs"]


def test_uniform_dist(port):
    assert port.uniform_dist(3).tolist() == [21846, 21845, 21845]  # test_coder.cpp:96-105
    assert set(port.uniform_dist(64).tolist()) == {1024}


def test_det_functions_match_reference(ref, port):
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-100, 100, 4000), rng.uniform(-3, 3, 4000), [0.0, -0.0, 87.5, -87.5]]).astype(np.float32)
    for which in range(4):
        xx = np.abs(x) + np.float32(1e-30) if which == 1 else x
        assert np.array_equal(ref.det(which, xx).view(np.uint32), port.det(which, xx).view(np.uint32))
    assert port.det(0, np.zeros(1, np.float32))[0] == 1.0  # test_detmath anchors
    assert port.det(2, np.zeros(1, np.float32))[0] == 0.5


def test_eq1_hand_value(port):
    # test_mixer.cpp:44-55: alpha=.5, lu=[2,0,0,0], lm=[0,2,0,0] -> softmax([1,1,0,0])
    p = port.softmax(np.array([1.0, 1.0, 0.0, 0.0], np.float32))
    assert np.allclose(p, [0.365529, 0.365529, 0.134471, 0.134471], atol=1e-6)


def test_containers_match_golden(port):
    import paper_2507_12805_b200 as P
    for case in json.loads((G / "containers.json").read_text()):
        raw = P.synth(case["gen"], case["n"], case["seed"]) if case["n"] else b""
        blob = port.compress(raw, O.make_cfg(**case["cfg"]))
        assert len(blob) == case["len"], case["name"]
        assert O.fnv1a64(blob) == case["fnv"], case["name"]
        assert port.decompress(blob) == raw, case["name"]


def test_port_matches_reference_spum_and_sprm(ref, port, spum_k3):
    import paper_2507_12805_b200 as P
    raw = P.synth("markov3", 30000, 5)
    c = O.make_cfg(t=8, bs=64, scale=16, workers=2, pub_path=spum_k3)
    a, sa = ref.compress(raw, c, with_stats=True)
    b, sb = port.compress(raw, c, with_stats=True)
    assert a == b and a[5] == 5  # flags = pub|dyn
    assert [x.snapshot_sent_hash for x in sa] == [x.snapshot_sent_hash for x in sb]
    assert [x.early_loss_bits for x in sa] == [x.early_loss_bits for x in sb]
    # SPrM branch (threshold 0 -> private model trained inside compress)
    raw2 = P.synth("markov3", 20000, 6) + b"NNacgt>\n"
    c2 = O.make_cfg(t=8, bs=64, scale=16, workers=2, threshold=0)
    a2 = ref.compress(raw2, c2)
    assert a2 == port.compress(raw2, c2) and a2[5] == 6
    assert port.decompress(a2) == raw2


def test_dump_probs_match_golden(port):
    z = np.load(G / "dump_k3_t8_bs16_s16.npz")
    pay, snap, probs = port.dump_chunk(z["tokens"], 4, 3, 8, 16, 16, 1234, max_steps=32)
    assert np.array_equal(probs.view(np.uint32), z["probs"].view(np.uint32))
    assert pay == z["payload"].tobytes()
    assert snap == z["snapshot"].tobytes()


def test_empty_container_golden_bytes(port):
    # test_container.cpp:50-70 writes a container with chosen seeds; compress of
    # empty input produces the same layout with W=0 (header + empty sections)
    blob = port.compress(b"", O.make_cfg())
    assert blob[:4] == b"PMKL" and blob[4] == 1 and int.from_bytes(blob[48:52], "little") == 0
    assert port.decompress(blob) == b""
