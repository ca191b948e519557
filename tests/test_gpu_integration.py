"""GPU: the drop-in, proven with the reference's own acceptance gauntlet
(tests/acceptance.cpp) built with integration/pipeline_b200.cpp in place of
the reference's core/src/pipeline.cpp and linked against libpmklc_b200.so
(integration/Makefile). Every compress/decompress/encode_chunk_standalone the
gauntlet makes -- 222 lossless round trips over window shapes, workers and
model branches (c1), entropy and learning rates (c4, c5), the snapshot
handoff (c7), the selector (c9), bit-identical reruns (c10) -- runs on the
B200; c2/c3/c6/c8 exercise the reference's own tokenizer, coder, metrics and
layers, which the binary links unchanged."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "integration" / "_build" / "acceptance_b200"


def test_reference_acceptance_gauntlet_through_b200():
    if not BIN.exists():
        pytest.skip("integration/_build/acceptance_b200 not built (needs /root/reference)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=1500,
                       cwd=str(BIN.parent))
    out = r.stdout
    print(out)
    for n in range(1, 11):
        assert f"criterion {n:2d} PASS" in out, (n, out[-3000:], r.stderr[-2000:])
    assert r.returncode == 0 and "all criteria passed" in out
