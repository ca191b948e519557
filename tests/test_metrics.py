"""CPU: Eq. 3-5 metrics against the reference's own test values
(tests/test_metrics.cpp:31-78) and per-block ratios of a reference container."""
import pytest

import oracles as O


def test_compression_ratio(P):
    # test_metrics.cpp:31-43
    assert P.compression_ratio(250, 1000) == pytest.approx(2.0)
    assert P.compression_ratio(1000, 1000) == pytest.approx(8.0)
    assert P.compression_ratio(0, 4096) == 0.0
    assert P.compression_ratio(123456, 1048576) == pytest.approx(123456.0 / 1048576.0 * 8.0)
    with pytest.raises(P.PmklcError) as e:
        P.compression_ratio(10, 0)
    assert e.value.errc == "EmptySource"


def test_throughput(P):
    # test_metrics.cpp:45-55
    assert P.throughput(1_000_000, 2.0, 2.0) == pytest.approx(250000.0)
    assert P.throughput(0, 1.0, 0.0) == 0.0
    assert P.throughput(4096, 0.5, 1.5) == pytest.approx(2048.0)
    with pytest.raises(P.PmklcError) as e:
        P.throughput(100, 0.0, 0.0)
    assert e.value.errc == "ZeroTime"


def test_robustness(P):
    # test_metrics.cpp:57-78: the paper's nine Table-4 values -> 4.45458 % (n-1)
    nine = [1.812, 1.943, 1.900, 1.850, 1.851, 1.651, 1.892, 1.866, 1.844]
    assert P.robustness(nine) == pytest.approx(4.45458, rel=5e-4)
    assert P.robustness([1.0, 3.0]) == pytest.approx(70.7106781)
    assert P.robustness([1.234]) == 0.0
    assert P.robustness([v * 1000.0 for v in nine]) == pytest.approx(P.robustness(nine))
    with pytest.raises(P.PmklcError) as e:
        P.robustness([])
    assert e.value.errc == "EmptyList"


def test_block_ratios_of_reference_container(P, checker):
    raw = checker.synth("genome", 60_000, 7, 3)
    blob = checker.compress(raw, O.make_cfg(t=8, bs=16, scale=16, workers=4))
    h = O.parse_container(blob)
    want = [(pl + trl) * 8.0 / ((tl - 1) * h["s"] + h["k"]) for (_, tl, _, pl, trl) in h["chunks"]]
    got = P.block_ratios(blob)
    assert got == pytest.approx(want, rel=1e-12)
    assert len(got) == 4
    # the CRP of those blocks
    assert P.robustness(got) >= 0.0
    # a flipped byte fails the container checksum like the reference reader
    bad = bytearray(blob)
    bad[len(bad) // 2] ^= 0x40
    with pytest.raises(P.PmklcError) as e:
        P.block_ratios(bytes(bad))
    assert e.value.errc == "ChecksumMismatch"


def test_synth_generators_identical(P, checker):
    # the checker library's copy of the generators (bench --impl reference)
    # produces the product's bytes
    for kind, n, seed, extra in [("genome", 300_001, 2025, 10), ("markov3", 5000, 12345, 0),
                                 ("species", 200_000, 3, 65536), ("uniform", 777, 9, 0)]:
        assert checker.synth(kind, n, seed, extra) == P.synth(kind, n, seed, extra), kind
