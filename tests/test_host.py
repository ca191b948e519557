"""CPU: the C-ABI library loads, exports every declared symbol, its host
logic (plan_chunks, snapshot_step, SMP schedule) matches the reference, and
compute entry points fail loudly (no CPU fallback) when no GPU is present."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    hdr = (ROOT / "include" / "pmklc_b200.h").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(pmklc_\w+)\s*\(", hdr)))


def test_exports_every_declared_symbol(P):
    L = P.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(P.EXPORTS)


def test_plan_chunks_reference_values(P, ref):
    # test_pipeline.cpp:53-97
    st, ln, bs, _ = P.plan_chunks(100, 4, 320, 32, 0)
    assert (st, ln, bs) == ([0], [100], 3)
    st, ln, bs, _ = P.plan_chunks(1000, 2, 1, 1, 0)
    assert (st, ln, bs) == ([0, 500], [500, 500], 1)
    st, ln, _, _ = P.plan_chunks(10, 3, 1, 1, 0)
    assert (st, ln) == ([0, 4, 7], [4, 3, 3])
    assert P.plan_chunks(0, 8, 320, 32, 500)[:3] == ([], [], 1)
    st, ln, bs, _ = P.plan_chunks(3, 2, 16, 4, 0)
    assert (ln, bs) == ([3], 1)
    # snapshot_step (test_pipeline.cpp:99-115)
    assert P.plan_chunks(1000, 1, 10, 1, 500)[3] == [5]
    assert P.plan_chunks(1000, 1, 10, 1, 501)[3] == [6]
    assert P.plan_chunks(1000, 1, 10, 1, 1)[3] == [1]
    # agreement with the reference over a sweep
    import itertools
    lib = ref.lib
    cap = 256
    A = (C.c_uint64 * cap)
    for m, w, bs, t, my in itertools.product([0, 1, 50, 349525, 10**7], [1, 3, 8, 256], [1, 16, 320],
                                             [1, 8, 32], [0, 1, 500, 9999]):
        s1, l1, n1 = A(), A(), A()
        cnt, bo = C.c_size_t(), C.c_uint32()
        assert lib.pmref_plan_chunks(C.c_uint64(m), w, bs, t, C.c_uint16(my), s1, l1, n1,
                                     C.c_size_t(cap), C.byref(cnt), C.byref(bo)) == 0
        st, ln, b2, sn = P.plan_chunks(m, w, bs, t, my)
        k = cnt.value
        assert (st, ln, b2) == (list(s1[:k]), list(l1[:k]), bo.value)
        assert sn == list(n1[:k])


def test_schedule_semantics(P):
    # chunk i+1 starts when chunk i reaches its snapshot step (pipeline.cpp:260-281)
    R, t = 16, 8
    lens = [16 * 100] * 4  # L = 100 batch steps, 92 model steps
    off, src, ss, ms, ticks = P.schedule(lens, R, t, 500)  # snap = ceil(5) = 5 <= t
    assert src == [-1, -1, -1, -1] and off == [0, 0, 0, 0] and ms == [92] * 4 and ticks == 92
    off, src, ss, ms, ticks = P.schedule(lens, R, t, 2000)  # snap = 20 -> 12 model steps
    assert src == [-1, 0, 1, 2] and ss == [0, 12, 12, 12] and off == [0, 12, 24, 36]
    assert ticks == 36 + 92
    off, src, ss, ms, ticks = P.schedule(lens, R, t, 0)  # SMP off: all independent
    assert src == [-1] * 4 and off == [0] * 4
    # a chunk too short to reach its snapshot forwards its inbound state
    lens2 = [16 * 100, 16 * 3, 16 * 100]
    off, src, ss, ms, ticks = P.schedule(lens2, R, t, 2000)
    assert src == [-1, 0, 0] and off[2] == off[1] == 12 and ms[1] == 0


def test_compute_fails_loudly_without_gpu(P):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.PmklcError) as e:
        P.compress(b"ACGT" * 100)
    assert e.value.errc == "CudaError"
    with pytest.raises(P.PmklcError):
        P.skmer_encode(bytes(100), 3, 3)


def test_config_validation_matches_reference(P):
    # CompressConfig::validate (pipeline.cpp:16-24): rejected before any device work
    bad = [dict(s=4, k=3), dict(k=9, s=1), dict(t=0), dict(t=4097), dict(bs=0), dict(workers=0),
           dict(workers=257), dict(smp_fraction=1.0), dict(smp_fraction=-0.1), dict(scale=3)]
    for kw in bad:
        with pytest.raises(P.PmklcError) as e:
            P.compress(b"ACGT", P.CompressConfig(**kw))
        assert e.value.errc == "ConfigInvalid", kw


@pytest.mark.parametrize("W,L,smp,world", [(128, 813, 500, 1), (256, 4069, 500, 1), (64, 300, 3000, 1),
                                           (256, 4069, 500, 4), (16, 40, 0, 1), (4096, 2543, 500, 8)])
def test_slots_by_concurrency(P, W, L, smp, world):
    """Device memory by chunks in flight (assign_slots): no two chunks whose
    lifetimes (first model tick .. last tick, extended to the handoff ticks at
    which they are the source) overlap share a slot, every handoff source is
    live at its copy, and the slot count is far below W once SMP staggers
    the chunks."""
    bs, t = 320, 32
    lens = [bs * L] * W
    off, src, ss, ms, ticks = P.schedule(lens, bs, t, smp)
    for rank in range(world):
        slot, n = P.schedule_slots(lens, bs, t, smp, rank, world)
        life = {}
        for c in range(W):
            mine = c % world == rank
            if ms[c] and mine:
                assert slot[c] >= 0
                life[c] = [off[c], off[c] + ms[c] - 1]
            else:
                assert slot[c] == -1
        for c in range(W):
            if src[c] >= 0 and ms[c] and src[c] in life:
                life[src[c]][1] = max(life[src[c]][1], off[c])
        by_slot = {}
        for c, (a, b) in life.items():
            by_slot.setdefault(slot[c], []).append((a, b))
        for iv in by_slot.values():
            iv.sort()
            for (a0, b0), (a1, b1) in zip(iv, iv[1:]):
                assert a1 > b0, "overlapping lifetimes share a slot"
        assert n == len(by_slot)
        # greedy by start tick is optimal: slots == peak number of live chunks
        ev = sorted([(a, 1) for a, _ in life.values()] + [(b + 1, -1) for _, b in life.values()],
                    key=lambda e: (e[0], e[1]))
        peak = cur = 0
        for _, d in ev:
            cur += d
            peak = max(peak, cur)
        assert n == peak
        if smp and L > 640:  # SMP staggers chunks: fewer slots than chunks
            assert n < len(life), (n, len(life))
