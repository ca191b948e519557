"""Profiling driver: one compress of the exact bench.py config-3 workload
(100 MB synthetic genome seed 2025, W=128, seeded SPuM + DM). Used under ncu
for the launch list of the bench's step (profiles/)."""
import sys
import tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_12805_b200 as P
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
raw = P.synth("genome", n, 2025, 10)
spum = str(Path(tempfile.mkdtemp()) / "spum.bin")
P.write_bigru(spum, 3, 32, 4, 0xACE3, layers=2)
cfg = P.CompressConfig(workers=128, pub_model_path=spum)
tm = P.Timing()
blob = P.compress(raw, cfg)
print(f"n={n} -> {len(blob)} B")
