"""BASELINE config 2: (s,k)-mer encoder sweep over 2^30 synthetic bases (packed
2-bit, 268,435,456 bytes, Rng(1)) on one B200. HBM-bound: algorithmic bytes
= ceil(n/4) read + 4*m written per launch. Prints one JSON line per pair and a
summary; spot-checks tokens against the oracle on a prefix."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np
import torch

import paper_2507_12805_b200 as P

PAIRS = [(1, 1), (1, 2), (2, 2), (1, 3), (2, 3), (3, 3), (1, 4), (2, 4), (3, 4), (4, 4), (1, 8), (8, 8)]


def main():
    nbases = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 30)
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    packed = P.synth("packed", nbases // 4, 1)
    d_in = torch.frombuffer(bytearray(packed), dtype=torch.uint8).cuda()
    out = torch.empty((nbases + 8), dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # parity spot check on a prefix against the oracle
    import oracles as O
    chk = O.ref() if O.REF_SO.exists() else O.port()
    pre = np.frombuffer(packed[: 1 << 16], np.uint8)
    codes = np.unpackbits(pre[:, None], axis=1, bitorder="little")
    codes = (codes[:, 0::2] | (codes[:, 1::2] << 1)).reshape(-1).astype(np.uint8).tobytes()
    out16 = torch.empty((nbases + 16), dtype=torch.int16, device="cuda")
    results = []
    for s, k in PAIRS:
        m = (nbases - k) // s + 1
        want, _ = chk.skmer_encode(codes, s, k)
        for tw in (4, 2):  # u32 (the reference layout) and u16 tokens
            buf = out if tw == 4 else out16
            run = lambda: P.skmer_encode_packed_device(d_in.data_ptr(), nbases, s, k, buf.data_ptr(),
                                                       u16=(tw == 2))
            run()
            torch.cuda.synchronize()
            got = buf[: len(want)].cpu().numpy().view(np.uint32 if tw == 4 else np.uint16)
            ok = bool(np.array_equal(got.astype(np.uint32), want))
            ts = []
            for _ in range(iters):
                flush.add_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            byts = (nbases + 3) // 4 + tw * m
            gbs = byts / (ms / 1e3) / 1e9
            r = {"s": s, "k": k, "token_bytes": tw, "tokens": m, "ms": ms, "GB/s": gbs,
                 "frac": gbs / peak, "bases_per_s": nbases / (ms / 1e3), "parity_prefix_ok": ok}
            results.append(r)
            print(json.dumps(r), flush=True)
    print(json.dumps({"summary": "tokenizer sweep", "n_bases": nbases, "peak_gbs": peak,
                      "mean_frac_u32": sum(r["frac"] for r in results if r["token_bytes"] == 4)
                      / max(1, sum(1 for r in results if r["token_bytes"] == 4)),
                      "mean_frac_u16": sum(r["frac"] for r in results if r["token_bytes"] == 2)
                      / max(1, sum(1 for r in results if r["token_bytes"] == 2)),
                      "all_parity_ok": all(r["parity_prefix_ok"] for r in results)}))


if __name__ == "__main__":
    main()
