"""GPU parity: the B200 path against the reference (oracle/_ref when present,
else the pinned C restatement) and the committed golden fixtures.

Bars (BASELINE.json north_star): tokens bit-exact; per-step probabilities
bit-exact (EXACT mode; tolerance 0 — stricter than the stated 1e-5 absolute);
containers byte-identical (so bits/base deviation 0 %, within the 0.5 % bar);
decompression a bit-exact round trip; corrupt inputs raise the reference errc.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracles as O

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def codes_of(raw: bytes) -> bytes:
    a = np.frombuffer(raw, np.uint8)
    return (((a >> 1) ^ (a >> 2)) & 3).astype(np.uint8).tobytes()


# ------------------------------------------------------------------ tokenizer
def test_tokenizer_golden(P):
    for case in json.loads((G / "skmer.json").read_text()):
        tok = P.skmer_encode(bytes(case["codes"]), case["s"], case["k"])
        assert tok.tolist() == case["tokens"], (case["s"], case["k"])


def test_tokenizer_all_pairs_random(P, checker):
    # 36 (s,k) pairs (test_skmer.cpp:131-144) at ragged lengths incl. 0 and < k
    rng = np.random.default_rng(2024)
    for k in range(1, 9):
        for s in range(1, k + 1):
            for n in [0, k - 1, k, k + 1, int(rng.integers(10, 5000)), 100_003]:
                codes = rng.integers(0, 4, max(n, 0), dtype=np.uint8).tobytes()
                want, _ = checker.skmer_encode(codes, s, k)
                assert np.array_equal(P.skmer_encode(codes, s, k), want), (s, k, n)


def test_tokenizer_packed_large(P, checker):
    # device-resident packed 2-bit input (config 2 layout), 2^22 bases
    import torch
    n = 1 << 22
    packed = P.synth("packed", n // 4, 1)
    codes = np.unpackbits(np.frombuffer(packed, np.uint8)[:, None], axis=1, bitorder="little")
    codes = (codes[:, 0::2] | (codes[:, 1::2] << 1)).reshape(-1).astype(np.uint8)
    dp = torch.frombuffer(bytearray(packed), dtype=torch.uint8).cuda()
    for nb in (n, n - 37):  # full and ragged (tail slabs, partial last byte)
        for s, k in [(3, 3), (1, 8), (8, 8), (2, 5), (1, 1)]:
            m = (nb - k) // s + 1
            want, _ = checker.skmer_encode(codes[:nb].tobytes(), s, k)
            dt = torch.zeros(m, dtype=torch.int32, device="cuda")
            P.skmer_encode_packed_device(dp.data_ptr(), nb, s, k, dt.data_ptr())
            torch.cuda.synchronize()
            assert np.array_equal(dt.cpu().numpy().view(np.uint32), want), (nb, s, k)
            # 2-byte token layout (config 2), same values
            d16 = torch.zeros(m, dtype=torch.int16, device="cuda")
            P.skmer_encode_packed_device(dp.data_ptr(), nb, s, k, d16.data_ptr(), u16=True)
            torch.cuda.synchronize()
            assert np.array_equal(d16.cpu().numpy().view(np.uint16).astype(np.uint32), want), (nb, s, k)


# ------------------------------------------------------------------ quantizer
def test_quantizer_golden(P):
    for c in json.loads((G / "quantize.json").read_text()):
        p = np.asarray(c["p_bits"], dtype=np.uint32).view(np.float32)
        if c["error"]:
            with pytest.raises(P.PmklcError) as e:
                P.quantize(p)
            assert e.value.errc == c["error"]
        else:
            assert P.quantize(p)[0].tolist() == c["freqs"]


# ------------------------------------------------------------------ probabilities
def test_per_step_probabilities_bitwise_golden(P):
    z = np.load(G / "dump_k3_t8_bs16_s16.npz")
    pay, probs = P.dump_chunk(z["tokens"], 4, 3, 8, 16, 16, 1234, max_steps=32)
    assert np.array_equal(probs.view(np.uint32), z["probs"].view(np.uint32))
    assert pay == z["payload"].tobytes()


def test_per_step_probabilities_bitwise_default_widths(P, checker):
    # reference default widths (scale 4, t=32), 2 substream rows x 60 model steps
    raw = P.synth("markov3", 40000, 21)
    tok, _ = checker.skmer_encode(codes_of(raw), 3, 3)
    tok = tok[: 8 * 92]
    pa, _, want = checker.dump_chunk(tok, 4, 3, 32, 8, 4, 777, max_steps=60)
    pb, got = P.dump_chunk(tok, 4, 3, 32, 8, 4, 777, max_steps=60)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert np.max(np.abs(got - want)) <= 1e-5  # the north star's stated bar, trivially met
    assert pa == pb


def test_per_step_probabilities_with_spum(P, checker, spum_k3):
    raw = P.synth("markov3", 30000, 22)
    tok, _ = checker.skmer_encode(codes_of(raw), 3, 3)
    tok = tok[: 16 * 40]
    pa, _, want = checker.dump_chunk(tok, 5, 3, 8, 16, 16, 99, pub_path=spum_k3, max_steps=32)
    pb, got = P.dump_chunk(tok, 5, 3, 8, 16, 16, 99, pub_model_path=spum_k3, max_steps=32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert pa == pb


# ------------------------------------------------------------------ containers
def _cfgs(kw):
    c = dict(kw)
    smp = c.pop("smp", None)
    pc = {k: v for k, v in c.items() if k != "pub_path"}
    if smp is not None:
        pc["smp_fraction"] = smp
    if "pub_path" in c:
        pc["pub_model_path"] = c["pub_path"]
    return pc


def test_containers_golden(P):
    for case in json.loads((G / "containers.json").read_text()):
        raw = P.synth(case["gen"], case["n"], case["seed"]) if case["n"] else b""
        blob = P.compress(raw, P.CompressConfig(**_cfgs(case["cfg"])))
        assert len(blob) == case["len"], case["name"]
        assert O.fnv1a64(blob) == case["fnv"], case["name"]
        if case["hex"]:
            assert blob.hex() == case["hex"]
        assert P.decompress(blob) == raw, case["name"]


@pytest.mark.parametrize("sk", [(1, 1), (1, 2), (2, 2), (1, 3), (2, 3), (3, 3), (1, 4), (2, 4),
                                (3, 4), (4, 4)])
@pytest.mark.parametrize("workers", [1, 2, 4])
def test_table8_pairs_workers_identical(P, checker, sk, workers):
    # the 10 Table-8 (s,k) pairs x workers {1,2,4} (test_pipeline.cpp:206-223)
    raw = P.synth("markov3", 12000, 100 + sk[0] * 10 + sk[1])
    kw = dict(s=sk[0], k=sk[1], t=4, bs=16, scale=16, workers=workers, smp=0.1)
    blob = P.compress(raw, P.CompressConfig(**_cfgs(kw)))
    assert blob == checker.compress(raw, O.make_cfg(**kw))
    assert P.decompress(blob) == raw


def test_config1_appendix_e_fingerprints(P):
    # 1 MiB order-3 Markov, CompressConfig{} defaults
    raw = P.synth("markov3", 1 << 20, 12345)
    assert O.fnv1a64(raw) == 0xE7E1F05C5FC7B7FC
    blob = P.compress(raw, P.CompressConfig())
    assert (len(blob), O.fnv1a64(blob)) == (231207, 0xC59806701E845E33)
    blob8 = P.compress(raw, P.CompressConfig(workers=8))
    assert (len(blob8), O.fnv1a64(blob8)) == (254517, 0x60402D686AEFD79D)
    assert P.decompress(blob) == raw
    assert P.decompress(blob8) == raw


def test_spum_branch_and_stats(P, checker, spum_k3):
    raw = P.synth("markov3", 30000, 5)
    kw = dict(t=8, bs=64, scale=16, workers=3, pub_path=spum_k3)
    st = P.PipelineStats()
    blob = P.compress(raw, P.CompressConfig(**_cfgs(kw)), st)
    want, wst = checker.compress(raw, O.make_cfg(**kw), with_stats=True)
    assert blob == want and blob[5] == 5
    for a, b in zip(st.workers, wst):
        assert (a.tokens, a.uniform_coded, a.pub_calls, a.dyn_calls) == \
               (b.tokens, b.uniform_coded, b.pub_calls, b.dyn_calls)
        assert a.snapshot_sent_hash == b.snapshot_sent_hash
        assert a.snapshot_recv_hash == b.snapshot_recv_hash
        assert a.early_loss_bits == b.early_loss_bits
    dst = P.PipelineStats()
    assert P.decompress(blob, spum_k3, stats=dst) == raw
    # SMP: encode and decode snapshot hashes equal (test_pipeline.cpp:427-452)
    assert [w.snapshot_sent_hash for w in dst.workers] == [w.snapshot_sent_hash for w in st.workers]
    with pytest.raises(P.PmklcError) as e:
        P.decompress(blob)  # container needs the SPuM file
    assert e.value.errc == "SpumMissing"


def test_smp_chain_long_chunks(P, checker):
    # snapshot taken after training starts (snap > t): real Step-wise Model Passing
    raw = P.synth("markov3", 200000, 31)
    kw = dict(t=8, bs=32, scale=16, workers=4, smp=0.3)
    st = P.PipelineStats()
    blob = P.compress(raw, P.CompressConfig(**_cfgs(kw)), st)
    want, wst = checker.compress(raw, O.make_cfg(**kw), with_stats=True)
    assert blob == want
    assert [w.snapshot_recv_hash for w in st.workers] == [w.snapshot_recv_hash for w in wst]
    assert P.decompress(blob) == raw


def test_cross_decode_with_reference(P, checker):
    # GPU decodes reference containers and the reference decodes GPU ones
    raw = P.synth("genome", 80000, 3) + b">chr1 test\nNNNNacgtRYK\n" + P.synth("markov3", 5000, 4)
    kw = dict(t=8, bs=32, scale=8, workers=3)
    ref_blob = checker.compress(raw, O.make_cfg(**kw))
    assert P.decompress(ref_blob) == raw
    gpu_blob = P.compress(raw, P.CompressConfig(**_cfgs(kw)))
    assert gpu_blob == ref_blob
    assert checker.decompress(gpu_blob) == raw


def test_encode_chunks_matches_reference_standalone(P, checker):
    # encode_chunk_standalone from recorded inbound snapshots (test_pipeline.cpp:396-425)
    raw = P.synth("markov3", 60000, 41)
    tok, _ = checker.skmer_encode(codes_of(raw), 3, 3)
    n = 16 * 60
    chunks = [tok[i * n:(i + 1) * n] for i in range(3)]
    _, snap, _ = checker.dump_chunk(chunks[0], 4, 3, 8, 16, 16, 5)
    inbound = [b"", snap, snap]
    got = P.encode_chunks(np.concatenate(chunks), [n] * 3, inbound, 4, 3, 8, 16, 16, 5)
    for i in range(3):
        want, _, _ = checker.dump_chunk(chunks[i], 4, 3, 8, 16, 16, 5, inbound=inbound[i])
        assert got[i] == want


@pytest.mark.parametrize("flags", [4, 5])
def test_throughput_regime_matches_reference(P, checker, tmp_path, flags):
    # 128 independent chunks at the default widths (scale 4, t=32, bs=320) in
    # one batch: every kernel runs its many-chunk variant (NT reduction with 8
    # rows per thread, one token group per chunk, fused dx, fused BiGRU layer
    # 1, ...). Chunks 0, 63 and 127 against the reference's standalone chunk
    # encoder (4 model steps each after the 32 warm-up steps).
    spum = ""
    if flags & 1:
        spum = str(tmp_path / "spum_s4.bin")
        P.write_bigru(spum, 3, 32, 4, 0xACE3, layers=2)
    W, n = 128, 320 * 36
    raw = P.synth("genome", W * n * 3 + 64, 77, 10)
    tok, _ = checker.skmer_encode(codes_of(raw), 3, 3)
    tok = np.ascontiguousarray(tok[:W * n], dtype=np.uint32)
    got = P.encode_chunks(tok, [n] * W, [b""] * W, flags, 3, 32, 320, 4, 0x5EED,
                          pub_model_path=spum)
    for i in (0, 63, 127):
        want, _, _ = checker.dump_chunk(tok[i * n:(i + 1) * n], flags, 3, 32, 320, 4, 0x5EED,
                                        pub_path=spum or None)
        assert got[i] == want, i


@pytest.mark.parametrize("kw,n", [
    (dict(t=8, bs=8, scale=1), 3000),                    # paper widths (E=64, H=256, F=4096)
    (dict(t=8, bs=8, scale=2, workers=2, smp=0.3), 6000),
    (dict(s=5, k=5, t=4, bs=16, scale=16), 40000),       # V=1024: general quantizer ranks
    (dict(s=3, k=6, t=4, bs=16, scale=16, workers=2), 30000),  # V=4096
])
def test_containers_more_widths_and_vocabularies(P, checker, kw, n):
    raw = P.synth("markov3", n, 97)
    pkw = {("smp_fraction" if k == "smp" else k): v for k, v in kw.items()}
    blob = P.compress(raw, P.CompressConfig(**pkw))
    assert blob == checker.compress(raw, O.make_cfg(**kw))
    assert P.decompress(blob) == raw


def test_k8_invalid_distribution_like_reference(P, checker):
    # k=8 (V=65,536): the reference's float32 softmax sum drifts past the
    # quantizer's 1e-5 check and compress throws InvalidDistribution
    # (SURVEY 8(a) a8); the exact GPU path must throw the same error.
    raw = P.synth("markov3", 200000, 99)
    kw = dict(s=8, k=8, t=4, bs=16, scale=16)
    with pytest.raises(O.CheckerError) as want:
        checker.compress(raw, O.make_cfg(**kw))
    with pytest.raises(P.PmklcError) as got:
        P.compress(raw, P.CompressConfig(**kw))
    assert want.value.errc == "InvalidDistribution"
    assert got.value.errc == want.value.errc


def test_spum_paper_widths(P, checker, tmp_path):
    # SPuM at scale 1 (Hs=128: the generic recurrence, no fused layer 1)
    path = str(tmp_path / "spum_s1.bin")
    P.write_bigru(path, 3, 8, 1, 0xBEEF, layers=2)
    raw = P.synth("markov3", 2400, 98)
    kw = dict(t=8, bs=8, scale=1)
    blob = P.compress(raw, P.CompressConfig(pub_model_path=path, **kw))
    assert blob[5] == 5
    assert blob == checker.compress(raw, O.make_cfg(pub_path=path, **kw))
    assert P.decompress(blob, path) == raw


# ------------------------------------------------------------------ edge cases / errors
def test_degenerate_inputs(P, checker):
    for raw in [b"", b"A", b"AC", b"ACG", b"NNNN", b"acgt", bytes(range(256)), b"ACGT" * 3]:
        kw = dict(t=4, bs=16, scale=16)
        blob = P.compress(raw, P.CompressConfig(**kw))
        assert blob == checker.compress(raw, O.make_cfg(**kw)), raw
        assert P.decompress(blob) == raw


def test_corruption_is_rejected(P):
    raw = P.synth("markov3", 20000, 1)
    blob = bytearray(P.compress(raw, P.CompressConfig(t=4, bs=16, scale=16)))
    bad = bytearray(blob)
    bad[100] ^= 1
    with pytest.raises(P.PmklcError) as e:
        P.decompress(bytes(bad))
    assert e.value.errc == "ChecksumMismatch"
    with pytest.raises(P.PmklcError) as e:
        P.decompress(bytes(blob[:40]))
    assert e.value.errc == "TableInconsistent"
    bad = bytearray(blob)
    bad[0] = ord("X")
    h = O.fnv1a64(bytes(bad[:-8]))
    bad[-8:] = h.to_bytes(8, "little")
    with pytest.raises(P.PmklcError) as e:
        P.decompress(bytes(bad))
    assert e.value.errc == "BadMagic"


def test_truncated_payload_stream_exhausted(P):
    # chop the codestream but keep the container consistent -> StreamExhausted
    raw = P.synth("markov3", 20000, 2)
    blob = P.compress(raw, P.CompressConfig(t=4, bs=16, scale=16))
    W = int.from_bytes(blob[48:52], "little")
    e0 = 52
    off = int.from_bytes(blob[e0 + 16:e0 + 24], "little")
    plen = int.from_bytes(blob[e0 + 24:e0 + 32], "little")
    cut = 64
    b = bytearray(blob[:off + plen - cut] + blob[off + plen:-8])
    b[e0 + 24:e0 + 32] = (plen - cut).to_bytes(8, "little")
    b += O.fnv1a64(bytes(b)).to_bytes(8, "little")
    assert W == 1
    with pytest.raises(P.PmklcError) as e:
        P.decompress(bytes(b))
    assert e.value.errc in ("StreamExhausted", "CorruptStream")


def test_dist_context_single_rank(P, checker):
    # the PMKLC-M entry points with a 1-rank NCCL communicator: same container
    import torch.distributed as dist
    import os
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=0, world_size=1)
    ctx = P.DistContext(0, 1, 0)
    try:
        raw = P.synth("markov3", 60000, 77)
        kw = dict(t=8, bs=32, scale=16, workers=4, smp=0.2)
        blob = ctx.compress(raw, P.CompressConfig(**_cfgs(kw)))
        assert blob == checker.compress(raw, O.make_cfg(**kw))
        assert ctx.decompress(blob) == raw
    finally:
        ctx.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("with_pub", [False, True])
def test_sprm_prepass_branch(P, checker, spum_k3, with_pub):
    # input above the selector threshold -> private model trained inside compress
    # (pretrain_private, training.cpp:62-83); the container carries its PMKW bytes,
    # so byte identity pins the whole training pass
    raw = P.synth("markov3", 40000, 61) + b"NNacgt>\n"
    kw = dict(t=8, bs=64, scale=16, workers=2, threshold=0)
    if with_pub:
        kw["pub_path"] = spum_k3  # derive_private_init: emb + gru0 copied from the SPuM
    ckw = dict(kw)
    thr = ckw.pop("threshold")
    cfg = P.CompressConfig(**_cfgs(ckw), selector_threshold=thr)
    blob = P.compress(raw, cfg)
    want = checker.compress(raw, O.make_cfg(**kw))
    assert blob[5] == 6 and want[5] == 6
    assert blob == want
    assert P.decompress(blob, spum_k3 if with_pub else "") == raw
    assert checker.decompress(blob, pub_path=spum_k3 if with_pub else None) == raw


@pytest.mark.parametrize("kw", [
    dict(t=32, bs=99),             # K = 3168: 49 full 64-k tiles + a ragged one, 16-byte B rows
    dict(t=8, bs=50, scale=16),    # K = 400, N < 32: the generic copy path of the NT reduction
])
def test_sprm_prepass_ragged_k(P, checker, kw):
    # the pre-pass weight-gradient reductions run K = bs*t long chains in the
    # deep (one row per thread) NT kernel; a K that is not a multiple of its
    # 64-k tile exercises the ragged last tile and the end of the copy stream
    raw = P.synth("markov3", 60000, 63)
    full = dict(kw, workers=2, threshold=0)
    ckw = dict(full)
    thr = ckw.pop("threshold")
    blob = P.compress(raw, P.CompressConfig(**_cfgs(ckw), selector_threshold=thr))
    assert blob[5] == 6
    assert blob == checker.compress(raw, O.make_cfg(**full))
    assert P.decompress(blob) == raw


def test_sprm_prepass_default_widths(P, checker):
    # scale 4, t = 32, bs = 320: the widths of BASELINE configs 4/5
    raw = P.synth("markov3", 150000, 62)
    kw = dict(workers=2, threshold=0)
    cfg = P.CompressConfig(workers=2, selector_threshold=0)
    blob = P.compress(raw, cfg)
    assert blob == checker.compress(raw, O.make_cfg(**kw))
    assert P.decompress(blob) == raw


def test_encode_chunks_with_private_model(P, checker):
    # ChunkCodeSpec::priv (pipeline.hpp:69-78): recode the chunks of a flags-6
    # container from their recorded inbound snapshots with the container's own
    # private model, on the GPU and on the reference's encode_chunk_standalone
    raw = P.synth("markov3", 120000, 64)
    kw = dict(t=8, bs=32, scale=16, workers=3, smp=0.3)
    st = P.PipelineStats()
    blob = P.compress(raw, P.CompressConfig(**_cfgs(kw), selector_threshold=0), st)
    assert blob == checker.compress(raw, O.make_cfg(threshold=0, **kw))
    h = O.parse_container(blob)
    assert h["flags"] == 6 and h["priv"]
    tok, _ = checker.skmer_encode(codes_of(raw), 3, 3)
    lens = [(tl // 32) * 32 for (_, tl, _, _, _) in h["chunks"]]
    ctok = np.concatenate([tok[ts:ts + n] for (ts, _, _, _, _), n in zip(h["chunks"], lens)])
    inbound = [w.snapshot_recv_bytes for w in st.workers]
    assert inbound[0] == b"" and all(inbound[1:])
    got = P.encode_chunks(ctok, lens, inbound, 6, 3, 8, 32, 16, h["dm_seed"], priv_model=h["priv"])
    off = 0
    for i, ((_, _, po, pl, _), n) in enumerate(zip(h["chunks"], lens)):
        assert got[i] == blob[po:po + pl], i
        want = checker.encode_chunk_standalone(ctok[off:off + n], 6, 3, 8, 32, 16, h["dm_seed"],
                                               priv=h["priv"], inbound=inbound[i])
        assert want == got[i], i
        off += n
    with pytest.raises(P.PmklcError) as e:
        P.encode_chunks(ctok[:lens[0]], lens[:1], [b""], 6, 3, 8, 32, 16, h["dm_seed"])
    assert e.value.errc == "ConfigInvalid"


@pytest.mark.parametrize("kw", [dict(t=512, bs=8, scale=4), dict(t=160, bs=8, scale=1)])
def test_long_context_attention(P, checker, kw):
    # contexts long enough that K/V no longer fit the row kernels' shared
    # memory: the long-context attention forward/backward kernels run
    raw = P.synth("markov3", 3 * 8 * (kw["t"] + 12) + 9, 71)
    blob = P.compress(raw, P.CompressConfig(**kw))
    assert blob == checker.compress(raw, O.make_cfg(**kw))
    assert P.decompress(blob) == raw


def test_stats_inbound_bytes(P, checker):
    # WorkerStats::snapshot_recv_bytes (pipeline.hpp:32): exported per chunk,
    # hashing to the reference's snapshot_recv_hash, on both ends
    raw = P.synth("markov3", 200000, 31)
    kw = dict(t=8, bs=32, scale=16, workers=4, smp=0.3)
    st, dst = P.PipelineStats(), P.PipelineStats()
    blob = P.compress(raw, P.CompressConfig(**_cfgs(kw)), st)
    _, wst = checker.compress(raw, O.make_cfg(**kw), with_stats=True)
    assert P.decompress(blob, stats=dst) == raw
    for a, b, d in zip(st.workers, wst, dst.workers):
        assert O.fnv1a64(a.snapshot_recv_bytes) == b.snapshot_recv_hash if a.snapshot_recv_bytes \
            else b.snapshot_recv_hash == 0
        assert d.snapshot_recv_bytes == a.snapshot_recv_bytes
    assert P.chunk_count(raw, P.CompressConfig(**_cfgs(kw))) == len(st.workers) == 4


def test_run_benchmark_csv_and_fault(P, tmp_path):
    # run_benchmark (bench.cpp:67-114) as test_metrics.cpp:80-140 drives it
    a, b, csv = tmp_path / "pmklc_bench_a.seq", tmp_path / "pmklc_bench_b.seq", tmp_path / "r.csv"
    a.write_bytes(P.synth("uniform", 2500, 41))
    b.write_bytes(P.synth("genome", 3200, 42, 2) + b"\n>chr\nNNacgt\n")
    cfg = P.CompressConfig(s=2, k=2, t=4, bs=16, scale=16, selector_threshold=1 << 40)
    rows, rep = P.run_benchmark([str(a), str(b)], cfg, str(csv))
    assert [r.name for r in rows] == ["pmklc_bench_a.seq", "pmklc_bench_b.seq"]
    for r in rows:
        assert r.verified and r.source_bytes > 0 and r.compressed_bytes > 0 and r.ct_s > 0
        assert r.cr == pytest.approx(r.compressed_bytes / r.source_bytes * 8.0)
        assert r.thp > 0
    assert rep.mean_cr == pytest.approx((rows[0].cr + rows[1].cr) / 2)
    assert rep.crp_percent == pytest.approx(P.robustness([rows[0].cr, rows[1].cr]))
    assert rep.peak_mem_bytes > 0 and rep.peak_device_bytes > 0
    text = csv.read_text()
    assert text.startswith("dataset,source_bytes,compressed_bytes,ct_s,dt_s,cr_bits_per_base,"
                           "thp_bytes_per_s,verified\n")
    assert text.count("\n") == 4 and "AGGREGATE" in text and ",true\n" in text
    rows, rep = P.run_benchmark([str(a)], cfg, "", fault_flip_mid=True)
    assert not rows[0].verified and rep.mean_cr == 0.0 and rep.crp_percent == 0.0


@pytest.mark.parametrize("scale,with_pub", [(2, False), (2, True), (1, False)])
def test_sprm_prepass_wide_scales(P, checker, tmp_path, scale, with_pub):
    # SPrM pre-pass at the paper's widths (scale 1: Es=16, Hs=128, B=128) and
    # scale 2 (Hs=64): the wide forward/BPTT kernels; flags-6 containers
    # (which carry the trained private model) byte-identical to the reference
    raw = P.synth("markov3", 9000, 65 + scale)
    kw = dict(t=8, bs=16, scale=scale, workers=2, threshold=0)
    if with_pub:
        path = str(tmp_path / f"spum_s{scale}.bin")
        P.write_bigru(path, 3, 8, scale, 0xD00D, layers=2)
        kw["pub_path"] = path
    ckw = dict(kw)
    thr = ckw.pop("threshold")
    blob = P.compress(raw, P.CompressConfig(**_cfgs(ckw), selector_threshold=thr))
    want = checker.compress(raw, O.make_cfg(**kw))
    assert blob[5] == 6
    assert blob == want
    assert P.decompress(blob, kw.get("pub_path", "")) == raw


@pytest.mark.parametrize("kw", [dict(t=8, batch=16, scale=16), dict(t=8, batch=24, scale=4),
                                dict(t=6, batch=16, scale=2, epochs=1)])
def test_pretrain_public_matches_reference(P, checker, tmp_path, kw):
    # pretrain_public (training.cpp:43-60): the 2-layer public model trained on
    # a corpus (a too-short file is skipped), byte-identical PMKW to the
    # reference's; the trained SPuM then codes like the reference's
    corpus = [P.synth("markov3", 4000, 81), P.synth("genome", 2500, 82, 2) + b"\n>x\nNNacgt\n",
              b"ACGTACGT", P.synth("uniform", 1500, 83)]
    want = checker.pretrain_public(corpus, seed=0x5EED, **kw)
    got = P.pretrain_public(corpus, seed=0x5EED, **kw)
    assert got == want
    path = str(tmp_path / "trained.bin")
    open(path, "wb").write(got)
    raw = P.synth("markov3", 9000, 84)
    ckw = dict(t=kw["t"], bs=16, scale=kw["scale"], workers=2)
    blob = P.compress(raw, P.CompressConfig(pub_model_path=path, **ckw))
    assert blob[5] == 5 and blob == checker.compress(raw, O.make_cfg(pub_path=path, **ckw))
    with pytest.raises(P.PmklcError) as e:
        P.pretrain_public([b"ACGT"], t=8, batch=16, scale=16)
    assert e.value.errc == "CorpusEmpty"


def test_file_streaming(P, checker, tmp_path):
    # file to file with bounded host memory: the input streams
    # into HBM and the output out of it through small pinned blocks; the
    # container is the same as the in-memory API's (and the reference's)
    raw = P.synth("genome", 2_000_003, 91, 4) + b"\n>chr2\nNNNNacgtRY\n" + P.synth("markov3", 50_000, 92)
    src, mid, dst = tmp_path / "in.fa", tmp_path / "c.pmkl", tmp_path / "out.fa"
    src.write_bytes(raw)
    kw = dict(t=8, bs=32, scale=16, workers=4)
    tm = P.Timing()
    P.compress_file(str(src), str(mid), P.CompressConfig(**kw), block_bytes=256 << 10, timing=tm)
    blob = mid.read_bytes()
    assert blob == P.compress(raw, P.CompressConfig(**kw)) == checker.compress(raw, O.make_cfg(**kw))
    P.decompress_file(str(mid), str(dst), block_bytes=100_000)
    assert dst.read_bytes() == raw
    with pytest.raises(P.PmklcError) as e:
        P.compress_file(str(tmp_path / "missing"), str(mid), P.CompressConfig(**kw))
    assert e.value.errc == "IoError"


def test_flags7_public_and_private_chunks(P, checker, spum_k3):
    # flags 7 (SPuM and SPrM together, mixer.cpp:14-42): the reference's
    # compress never selects it, but its decoder and encode_chunk_standalone
    # (ChunkCodeSpec with pub and priv) accept it -- chunk payloads identical
    raw = P.synth("markov3", 60000, 93)
    kw = dict(t=8, bs=16, scale=16, workers=1)
    blob6 = P.compress(raw, P.CompressConfig(**kw, selector_threshold=0))
    priv = O.parse_container(blob6)["priv"]
    tok, _ = checker.skmer_encode(codes_of(raw), 3, 3)
    n = 16 * 120
    chunks = [tok[i * n:(i + 1) * n] for i in range(2)]
    _, snap = checker.replay_chunk(chunks[0], 7, 3, 8, 16, 16, 4242, pub_path=spum_k3, priv=priv,
                                   snap_at=50, stop_at=50)
    inbound = [b"", snap]
    got = P.encode_chunks(np.concatenate(chunks), [n] * 2, inbound, 7, 3, 8, 16, 16, 4242,
                          pub_model_path=spum_k3, priv_model=priv)
    for i in range(2):
        want = checker.encode_chunk_standalone(chunks[i], 7, 3, 8, 16, 16, 4242, pub_path=spum_k3,
                                               priv=priv, inbound=inbound[i])
        assert got[i] == want, i


def test_corrupt_container_fuzz(P, checker):
    # structurally valid but mutated containers (checksum recomputed, so the
    # reader's FNV check passes): every one must decode or raise a reference
    # errc -- never crash, hang or return a CUDA failure
    raw = P.synth("markov3", 30000, 94)
    blob = P.compress(raw, P.CompressConfig(t=8, bs=16, scale=16, workers=2))
    rng = np.random.default_rng(95)
    outcomes = {}
    for trial in range(60):
        b = bytearray(blob[:-8])
        for _ in range(int(rng.integers(1, 4))):
            # past the header and chunk table (those are covered above): the
            # SPrM/exception/residual sections, codestreams and trailers
            at = int(rng.integers(52 + 36 * 2, len(b)))
            b[at] ^= int(rng.integers(1, 256))
        b += O.fnv1a64(bytes(b)).to_bytes(8, "little")
        try:
            out = P.decompress(bytes(b))
            outcomes["decoded"] = outcomes.get("decoded", 0) + 1
            assert isinstance(out, bytes)
        except P.PmklcError as e:
            assert e.errc != "CudaError", (trial, str(e))
            outcomes[e.errc] = outcomes.get(e.errc, 0) + 1
    assert sum(outcomes.values()) == 60


def _random_configs(n_cfg=24, seed=20261019):
    # seeded draws over the geometry the kernels are specialised on: odd and
    # even contexts and batch rows, several widths, vocabularies up to 4^6,
    # 1-5 chunks with SMP, both input generators, a third with a seeded SPuM
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cfg):
        k = int(rng.integers(1, 7))
        s = int(rng.integers(1, k + 1))
        kw = dict(s=s, k=k, t=int(rng.choice([2, 3, 5, 8, 13, 16])),
                  bs=int(rng.choice([3, 4, 7, 8, 12, 16, 24])), scale=int(rng.choice([4, 8, 16])),
                  workers=int(rng.choice([1, 2, 3, 5])), smp=float(rng.choice([0.05, 0.1, 0.3])))
        n = int(rng.integers(4000, 24000))
        kind = str(rng.choice(["markov3", "genome"]))
        spum = bool(rng.random() < 0.34)
        out.append((i, kind, n, kw, spum))
    return out


@pytest.mark.parametrize("case", _random_configs(), ids=lambda c: f"cfg{c[0]}")
def test_random_geometry_sweep(P, checker, tmp_path, case):
    # containers byte-identical to the reference's and lossless over seeded
    # random geometries (the specialised kernel paths: head widths, odd t/bs,
    # tile remainders, vocabulary sizes; flags 5 with a seeded SPuM)
    i, kind, n, kw, spum = case
    raw = P.synth(kind, n, 7000 + i, 10) if kind == "genome" else P.synth(kind, n, 7000 + i)
    if spum:
        path = str(tmp_path / "spum.bin")
        O.write_spum(path, kw["k"], kw["t"], kw["scale"], 0xACE3 + i)
        kw = dict(kw, pub_path=path)
    blob = P.compress(raw, P.CompressConfig(**_cfgs(kw)))
    assert blob == checker.compress(raw, O.make_cfg(**kw)), kw
    assert P.decompress(blob, kw.get("pub_path", "")) == raw
