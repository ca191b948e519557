"""GPU parity at benchmark scale, against goldens the reference itself produced
(tests/golden/make_bench_golden.py, run in the build container):

* the exact bench.py config-3 workload (100 MB synthetic genome, W=128 data
  blocks, SPuM + DM, defaults): the B200 container must be byte-identical to
  the reference's -- same length and FNV-1a, every chunk's payload, every
  chunk's inbound Step-wise Model Passing snapshot (WorkerStats
  snapshot_recv_hash; the bytes themselves are exported, pipeline.hpp:32) --
  and sampled chunks recoded on the GPU from their recorded inbound snapshots
  (encode_chunk_standalone, test_pipeline.cpp:396-425) reproduce their payloads;
* the SPrM pre-pass on a 3.2 MB prefix at the default widths (> 3,000
  strictly sequential Adam steps, warm-started from the SPuM): the private
  model blob and the flags-6 container are byte-identical.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracles as O

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def _golden(name):
    p = G / name
    if not p.exists():
        pytest.skip(f"{p.name} not generated (tests/golden/make_bench_golden.py)")
    return json.loads(p.read_text())


def _fnv(P, b):
    return f"{P.fnv1a64(b):016x}"


def test_bench_config3_container_identical_to_reference(P, tmp_path):
    g = _golden("bench_config3.json")
    raw = P.synth("genome", 100_000_000, 2025, 10)
    spum = str(tmp_path / "spum_k3_t32_s4.bin")
    assert f"{P.write_bigru(spum, 3, 32, 4, 0xACE3, layers=2):016x}" == g["spum_fingerprint"]
    st = P.PipelineStats()
    blob = P.compress(raw, P.CompressConfig(workers=128, pub_model_path=spum), st)
    h = O.parse_container(blob)
    assert h["flags"] == g["flags"] == 5
    assert len(h["chunks"]) == len(g["chunks"]) == 128
    for i, ((ts, tl, po, pl, _), want, w) in enumerate(zip(h["chunks"], g["chunks"], st.workers)):
        assert (ts, tl, pl) == (want["token_start"], want["token_len"], want["payload_len"]), i
        assert _fnv(P, blob[po:po + pl]) == want["payload_fnv"], i
        assert f"{w.snapshot_recv_hash:016x}" == want["recv_hash"], i
        assert f"{w.snapshot_sent_hash:016x}" == want["sent_hash"], i
        assert w.early_loss_bits == pytest.approx(want["early_loss_bits"], rel=0, abs=0), i
        if i:  # the exported inbound bytes are the snapshot the hash names
            assert _fnv(P, w.snapshot_recv_bytes) == want["recv_hash"], i
    assert (len(blob), _fnv(P, blob)) == (g["container_len"], g["container_fnv"])
    # encode_chunk_standalone from the recorded inbound snapshots (SURVEY 8(c)
    # parity protocol step 5) on the GPU: sampled chunks reproduce their payloads
    codes = np.frombuffer(raw, np.uint8)
    tok = P.skmer_encode((((codes >> 1) ^ (codes >> 2)) & 3).astype(np.uint8).tobytes(), 3, 3)
    picks = (1, 63, 127)
    L = [h["chunks"][i][1] // 320 for i in picks]
    ctok = np.concatenate([tok[h["chunks"][i][0]:h["chunks"][i][0] + 320 * l]
                           for i, l in zip(picks, L)])
    got = P.encode_chunks(ctok, [320 * l for l in L], [st.workers[i].snapshot_recv_bytes for i in picks],
                          5, 3, 32, 320, 4, h["dm_seed"], pub_model_path=spum)
    for i, pay in zip(picks, got):
        _, _, po, pl, _ = h["chunks"][i]
        assert pay == blob[po:po + pl], i
    # and the decoder reproduces the input
    assert P.decompress(blob, spum) == raw


def test_sprm_prepass_3mb_prefix_identical_to_reference(P, tmp_path):
    g = _golden("bench_sprm_prefix.json")
    raw = P.synth("genome", 100_000_000, 2025, 10)[:3_200_000]
    spum = str(tmp_path / "spum_k3_t32_s4.bin")
    P.write_bigru(spum, 3, 32, 4, 0xACE3, layers=2)
    cfg = P.CompressConfig(workers=4, selector_threshold=0, pub_model_path=spum)
    blob = P.compress(raw, cfg)
    h = O.parse_container(blob)
    assert h["flags"] == g["flags"] == 6
    assert g["train_steps"] >= 3000
    assert (len(h["priv"]), _fnv(P, h["priv"])) == (g["sprm_blob_len"], g["sprm_blob_fnv"])
    assert [_fnv(P, blob[po:po + pl]) for (_, _, po, pl, _) in h["chunks"]] == g["payload_fnv"]
    assert (len(blob), _fnv(P, blob)) == (g["container_len"], g["container_fnv"])
    assert P.decompress(blob, spum) == raw
