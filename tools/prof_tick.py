"""Profiling driver: one compress of SURVEY config 1 (1 MiB order-3 Markov,
defaults, W=1) or a multi-chunk variant. Used under ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_12805_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 20)
w = int(sys.argv[2]) if len(sys.argv) > 2 else 1
raw = P.synth("markov3", n, 12345)
st = P.PipelineStats()
blob = P.compress(raw, P.CompressConfig(workers=w), st)
t = st.timing
print(f"n={n} W={w} -> {len(blob)} B; total {t.total_ms:.1f} ms model {t.model_ms:.1f} ms ticks {t.ticks} launches {t.kernel_launches}")
