"""Profiling driver: compress with the SPrM branch (selector threshold 0)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_12805_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
raw = P.synth("genome", n, 5, 10)
st = P.PipelineStats()
b = P.compress(raw, P.CompressConfig(workers=4, selector_threshold=0), st)
print("flags", b[5], "launches", st.timing.kernel_launches, "total_ms", round(st.timing.total_ms, 1))
