"""Regenerate tests/golden/* from the REFERENCE (oracle/_ref/libpmklc_ref.so,
compiled from /root/reference/proj/core/src by oracle/Makefile).

Run here (the container that has /root/reference):  python tests/golden/make_golden.py
The fixtures let the GPU tests check parity even where oracle/_ref is absent.
Inputs are regenerated from seeds by paper_2507_12805_b200.synth (a pure
integer/IEEE generator, same bytes on any host) or numpy's PCG64 with fixed
seeds, and stored alongside for self-containment.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracles as O  # noqa: E402
import paper_2507_12805_b200 as P  # noqa: E402

R = O.ref()


def skmer_cases():
    rng = np.random.default_rng(2024)
    out = [{"s": 3, "k": 3, "codes": [1, 2, 2], "tokens": [26], "residual": []}]  # test_skmer.cpp:38-43
    for k in range(1, 9):
        for s in range(1, k + 1):
            n = int(rng.integers(0, 300))
            codes = rng.integers(0, 4, n, dtype=np.uint8)
            tok, res = R.skmer_encode(codes.tobytes(), s, k)
            out.append({"s": s, "k": k, "codes": codes.tolist(), "tokens": tok.tolist(),
                        "residual": list(res)})
    return out


def quantize_cases():
    # frozen vectors from test_coder.cpp:53-70 plus reference outputs on
    # random / skewed / clamped rows (incl. surplus cases that need several
    # sweep passes, coder.cpp:67-83)
    rows = [
        [0.97, 0.01, 0.01, 0.01], [0.9999985, 5e-7, 5e-7, 5e-7], [0.25] * 4,
        [0.4, 0.3, 0.2, 0.1], [np.float32(1.0) / np.float32(3), np.float32(1.0) / np.float32(3),
                               np.float32(1.0) / np.float32(3) + np.float32(1e-7)],
    ]
    rng = np.random.default_rng(77)
    for i in range(300):
        V = int(rng.choice([2, 3, 4, 16, 64, 100, 256, 1024]))
        kind = i % 4
        u = rng.random(V, dtype=np.float32) + np.float32(1e-4)
        if kind == 1:
            u = u ** 4
        elif kind == 2:
            u = np.exp(np.float32(20.0) * u).astype(np.float32)
        elif kind == 3:
            u = np.full(V, np.float32(1e-7), dtype=np.float32)
            u[rng.integers(0, V)] = np.float32(1.0)
        p = (u / u.astype(np.float64).sum()).astype(np.float32)
        # float renormalisation like the reference test helper (test_coder.cpp:28-50)
        fs = np.float32(0)
        for v in p:
            fs = np.float32(fs + v)
        j = int(np.argmax(p))
        p[j] = np.float32(p[j] + (np.float32(1.0) - fs))
        rows.append(p.tolist())
    cases = []
    for r in rows:
        p = np.asarray(r, dtype=np.float32)
        try:
            f = R.quantize(p).tolist()
            err = None
        except O.CheckerError as e:
            f, err = None, e.errc
        cases.append({"p_bits": p.view(np.uint32).tolist(), "freqs": f, "error": err})
    return cases


CONTAINER_CASES = [
    # (name, generator, n, seed, cfg)
    ("uniform_t4096", "uniform", 12000, 9, dict(t=4096)),
    ("uniform_t4096_res", "uniform", 12002, 9, dict(t=4096)),
    ("w1_small", "markov3", 20000, 1, dict(t=4, bs=16, scale=16)),
    ("w3_smp", "markov3", 50000, 2, dict(t=8, bs=64, scale=16, workers=3)),
    ("k1_w2", "markov3", 20000, 5, dict(s=1, k=1, t=4, bs=16, scale=16, workers=2, smp=0.1)),
    ("k4_s2", "markov3", 20000, 6, dict(s=2, k=4, t=4, bs=16, scale=16, workers=2, smp=0.1)),
    ("k2_s1_w4", "markov3", 30000, 11, dict(s=1, k=2, t=8, bs=32, scale=16, workers=4, smp=0.2)),
    ("smp_off_w4", "markov3", 40000, 12, dict(t=8, bs=32, scale=16, workers=4, smp=0.0)),
    ("tiny", "markov3", 50, 13, dict(t=4, bs=16, scale=16)),
    ("empty", "markov3", 0, 13, dict()),
    ("scale8_t16", "markov3", 60000, 14, dict(t=16, bs=48, scale=8, workers=2)),
]


def container_cases():
    out = []
    for name, gen, n, seed, kw in CONTAINER_CASES:
        raw = P.synth(gen, n, seed) if n else b""
        blob = R.compress(raw, O.make_cfg(**kw))
        out.append({"name": name, "gen": gen, "n": n, "seed": seed, "cfg": kw,
                    "len": len(blob), "fnv": O.fnv1a64(blob),
                    "hex": blob.hex() if len(blob) <= 4096 else None})
    return out


def dump_case():
    raw = P.synth("markov3", 30000, 3)
    codes = bytes(((b >> 1) ^ (b >> 2)) & 3 for b in raw)
    tok, _ = R.skmer_encode(codes, 3, 3)
    tok = tok[: 16 * 40]
    pay, snap, probs = R.dump_chunk(tok, 4, 3, 8, 16, 16, 1234, max_steps=32)
    np.savez_compressed(HERE / "dump_k3_t8_bs16_s16.npz", tokens=tok, probs=probs,
                        payload=np.frombuffer(pay, np.uint8), snapshot=np.frombuffer(snap, np.uint8))


def main():
    (HERE / "skmer.json").write_text(json.dumps(skmer_cases()))
    (HERE / "quantize.json").write_text(json.dumps(quantize_cases()))
    (HERE / "containers.json").write_text(json.dumps(container_cases(), indent=0))
    dump_case()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
