"""Compare the GEMM tile variants built by gemm_variants.sh: the gemm_ffn
microbenchmark and a 20 MB SPuM+DM compress (model ms), one subprocess per
variant library. Containers must hash identically (the ring depth does not
change any reduction order)."""
import hashlib
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
LIBDIR = ROOT / "paper_2507_12805_b200" / "lib"

CHILD = r'''
import sys, json, hashlib, time
sys.path.insert(0, %r)
from pathlib import Path
import paper_2507_12805_b200 as P
P.LIB_PATH = Path(%r)
import torch
out = {}
for ch in (87, 128):
    ms, fl, _ = P.bench_kernel("gemm_ffn", ch, iters=50)
    out["ffn_%%d_us" %% ch] = ms * 1e3
n = %d
raw = P.synth("genome", n, 2026, 10)
d = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
cfg = P.CompressConfig(workers=128, pub_model_path=%r)
best = 1e30
for rep in range(3):
    tc = P.Timing()
    blob = P.compress_device(d.data_ptr(), n, cfg, tc)
    best = min(best, tc.model_ms)
out["compress_model_ms"] = best
out["sha"] = hashlib.sha256(blob).hexdigest()[:16]
# SPrM pre-pass (the NT launch's deep, latency regime): 10^6 bases, flags 6
d6 = d[:1_000_000]
cfg6 = P.CompressConfig(workers=128, selector_threshold=0)
best6 = 1e30
for rep in range(3):
    tc = P.Timing()
    blob6 = P.compress_device(d6.data_ptr(), 1_000_000, cfg6, tc)
    best6 = min(best6, tc.sprm_ms)
out["sprm_ms"] = best6
out["sha6"] = hashlib.sha256(blob6).hexdigest()[:16]
print("RESULT " + json.dumps(out))
'''

def main():
    n = int(float(sys.argv[1]) * 1e6) if len(sys.argv) > 1 else 20_000_000
    spum = "/tmp/spum_k3.bin"
    sys.path.insert(0, str(ROOT))
    import paper_2507_12805_b200 as P
    P.write_bigru(spum, 3, 32, 4, 0xACE3)
    for so in sorted(LIBDIR.glob("var_*.so")):
        r = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), str(so), n, spum)],
                           capture_output=True, text=True, timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        res = json.loads(line[0][7:]) if line else {"error": r.stderr[-400:]}
        res["variant"] = so.stem
        print(json.dumps(res), flush=True)

main()
