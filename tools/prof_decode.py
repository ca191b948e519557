"""Profiling driver: decompress of a flags-6 container (selector threshold 0)
at W blocks; used under ncu for the decode-path kernels.
Usage: python tools/prof_decode.py [N_BYTES] [W]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_12805_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 8
raw = P.synth("genome", n, 2026, 10)
blob = P.compress(raw, P.CompressConfig(workers=w, selector_threshold=0))
assert P.decompress(blob) == raw
print("ok", len(raw), len(blob))
