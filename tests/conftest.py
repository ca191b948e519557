import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: longer oracle comparisons")


@pytest.fixture(scope="session")
def ref():
    import oracles
    if not oracles.REF_SO.exists():
        pytest.skip("oracle/_ref/libpmklc_ref.so not built (needs /root/reference at build time)")
    return oracles.ref()


@pytest.fixture(scope="session")
def port():
    import oracles
    if not oracles.PORT_SO.exists():
        import subprocess
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "port"], check=True)
    return oracles.port()


@pytest.fixture(scope="session")
def checker():
    """The reference itself when built, else the (pinned) C restatement."""
    import oracles
    if oracles.REF_SO.exists():
        return oracles.ref()
    if not oracles.PORT_SO.exists():
        import subprocess
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "port"], check=True)
    return oracles.port()


@pytest.fixture(scope="session")
def P():
    import paper_2507_12805_b200 as pkg
    pkg.lib()
    return pkg


@pytest.fixture(scope="session")
def spum_k3(tmp_path_factory, checker):
    """Seeded, untrained SPuM file (acceptance.cpp:58-69), t=8, scale 16.

    Written with the reference when present, else with the port's writer path
    via a committed fixture."""
    import oracles
    path = tmp_path_factory.mktemp("spum") / "spum_k3_t8_s16.bin"
    golden = ROOT / "tests" / "golden" / "spum_k3_t8_s16.bin"
    if oracles.REF_SO.exists():
        oracles.write_spum(str(path), 3, 8, 16, 0xACE3)
    else:
        path.write_bytes(golden.read_bytes())
    return str(path)
