"""Profiling driver: compress with the SPrM branch (selector threshold 0)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_12805_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
raw = P.synth("genome", n, 5, 10)
st = P.PipelineStats()
b = P.compress(raw, P.CompressConfig(workers=4, selector_threshold=0), st)
t = st.timing
print("flags", b[5], "launches", t.kernel_launches, "total_ms", round(t.total_ms, 1), "sprm_ms",
      round(t.sprm_ms, 1), "model_ms", round(t.model_ms, 1))
