"""Profiling driver: one compress of SURVEY config 1 (1 MiB order-3 Markov,
defaults, W=1) or a multi-chunk variant. Used under ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_12805_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 20)
w = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spum = len(sys.argv) > 3 and sys.argv[3] == "spum"
raw = P.synth("markov3", n, 12345)
cfg = P.CompressConfig(workers=w)
if spum:
    P.write_bigru("/tmp/prof_spum.bin", 3, 32, 4, 0xACE3)
    cfg.pub_model_path = "/tmp/prof_spum.bin"
st = P.PipelineStats()
blob = P.compress(raw, cfg, st)
t = st.timing
print(f"n={n} W={w} -> {len(blob)} B; total {t.total_ms:.1f} ms model {t.model_ms:.1f} ms ticks {t.ticks} launches {t.kernel_launches}")
