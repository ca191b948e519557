"""pmklc_b200 — B200-native PMKLC compress/decompress hot path.

Python mirror of the reference's public API (core/include/pmklc/pipeline.hpp):
``CompressConfig`` with the same fields and defaults, ``compress`` /
``decompress`` with the same argument meaning, ``PmklcError`` carrying the
reference ``errc`` name (core/include/pmklc/error.hpp). Every call goes
through the C ABI in include/pmklc_b200.h (lib/libpmklc_b200.so, built in-tree
by ``__graft_entry__.build()``); there is no CPU fallback — if the library or
a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional, Sequence

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "lib" / "libpmklc_b200.so"

ERRC = [
    "LengthMismatch", "TokenOutOfRange", "NotOverlapping", "ShapeMismatch", "StaleTape",
    "ContextLengthMismatch", "ChecksumMismatch", "ArchitectureMismatch", "MissingLogits",
    "BatchMismatch", "InvalidDistribution", "StreamExhausted", "BadMagic", "UnsupportedVersion",
    "TableInconsistent", "ConfigInvalid", "IoError", "SpumMissing", "CorruptStream", "CorpusEmpty",
    "TargetTooShort", "EmptySource", "ZeroTime", "EmptyList", "VerificationFailed",
]


class PmklcError(RuntimeError):
    """pmklc::error equivalent: ``.errc`` is the reference enum name."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.errc = ERRC[code - 1] if 1 <= code <= len(ERRC) else ("CudaError" if code == 101 else "Unknown")
        super().__init__(message)


class _Cfg(C.Structure):
    _fields_ = [("s", C.c_uint32), ("k", C.c_uint32), ("t", C.c_uint32), ("bs", C.c_uint32),
                ("workers", C.c_uint32), ("scale", C.c_uint32),
                ("selector_threshold", C.c_uint64), ("seed", C.c_uint64),
                ("smp_fraction", C.c_float), ("pub_model_path", C.c_char_p),
                ("device", C.c_int32), ("max_workers", C.c_uint32)]


class Stats(C.Structure):
    """pmklc_stats: WorkerStats (pipeline.hpp:27-35), one per chunk."""
    _fields_ = [("tokens", C.c_uint64), ("uniform_coded", C.c_uint64), ("pub_calls", C.c_uint64),
                ("priv_calls", C.c_uint64), ("dyn_calls", C.c_uint64),
                ("snapshot_recv_hash", C.c_uint64), ("snapshot_sent_hash", C.c_uint64),
                ("snapshot_recv_bytes", C.POINTER(C.c_uint8)), ("snapshot_recv_len", C.c_uint64),
                ("early_loss_bits", C.c_double)]


@dataclass
class WorkerStats:
    """pmklc::WorkerStats (pipeline.hpp:27-35); snapshot_recv_bytes is the
    chunk's inbound SMP snapshot (empty: seeded init), as the reference keeps
    it when stats are collected (pipeline.cpp:108-111)."""
    tokens: int = 0
    uniform_coded: int = 0
    pub_calls: int = 0
    priv_calls: int = 0
    dyn_calls: int = 0
    snapshot_recv_hash: int = 0
    snapshot_sent_hash: int = 0
    snapshot_recv_bytes: bytes = b""
    early_loss_bits: float = 0.0


def _worker_stats(st, n: int) -> List[WorkerStats]:
    out = []
    for i in range(n):
        e = st[i]
        b = C.string_at(e.snapshot_recv_bytes, e.snapshot_recv_len) if e.snapshot_recv_len else b""
        out.append(WorkerStats(e.tokens, e.uniform_coded, e.pub_calls, e.priv_calls, e.dyn_calls,
                               e.snapshot_recv_hash, e.snapshot_sent_hash, b, e.early_loss_bits))
    lib().pmklc_stats_release(st, C.c_size_t(n))
    return out


class Timing(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("h2d_ms", C.c_double), ("tokenize_ms", C.c_double),
                ("warmup_ms", C.c_double), ("model_ms", C.c_double), ("d2h_ms", C.c_double),
                ("ticks", C.c_uint64), ("kernel_launches", C.c_uint64), ("chunks", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("hot_ms", C.c_double), ("hot_launches", C.c_uint64), ("hot_units", C.c_uint64),
                ("hot_flops_per_unit", C.c_double), ("sprm_ms", C.c_double),
                ("slots", C.c_uint64), ("dev_peak_bytes", C.c_uint64)]


# Every symbol include/pmklc_b200.h declares (checked by tests/test_host.py).
EXPORTS = [
    "pmklc_cfg_default", "pmklc_compress", "pmklc_compress_device", "pmklc_decompress",
    "pmklc_decompress_to_device", "pmklc_encode_chunks", "pmklc_dump_chunk", "pmklc_skmer_encode",
    "pmklc_skmer_encode_packed_device", "pmklc_skmer_encode_packed_device_u16", "pmklc_free", "pmklc_device_free", "pmklc_last_error",
    "pmklc_errc_name", "pmklc_version", "pmklc_synth_markov3", "pmklc_synth_uniform",
    "pmklc_synth_genome", "pmklc_synth_species", "pmklc_synth_packed_codes", "pmklc_plan_chunks",
    "pmklc_schedule", "pmklc_quantize", "pmklc_write_bigru", "pmklc_bench_kernel",
    "pmklc_nccl_id", "pmklc_dist_create", "pmklc_dist_destroy", "pmklc_compress_dist",
    "pmklc_decompress_dist", "pmklc_dist_plan", "pmklc_stats_release", "pmklc_chunk_count",
    "pmklc_container_chunks", "pmklc_decompress_dist_to_device", "pmklc_compression_ratio",
    "pmklc_throughput", "pmklc_robustness", "pmklc_block_ratios", "pmklc_run_benchmark",
    "pmklc_fnv1a64", "pmklc_cfg_validate", "pmklc_schedule_slots", "pmklc_pretrain_public",
    "pmklc_compress_file", "pmklc_decompress_file",
]

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree C ABI library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        L = C.CDLL(str(LIB_PATH))
        L.pmklc_last_error.restype = C.c_char_p
        L.pmklc_errc_name.restype = C.c_char_p
        L.pmklc_version.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise PmklcError(rc, lib().pmklc_last_error().decode(errors="replace"))


def _take(ptr, n: int) -> bytes:
    b = C.string_at(ptr, n)
    lib().pmklc_free(ptr)
    return b


@dataclass
class CompressConfig:
    """pmklc::CompressConfig (pipeline.hpp:12-25), same defaults."""
    s: int = 3
    k: int = 3
    t: int = 32
    bs: int = 320
    workers: int = 1
    selector_threshold: int = 500_000_000
    smp_fraction: float = 0.05
    seed: int = 42
    scale: int = 4
    pub_model_path: str = ""
    device: int = 0
    max_workers: int = 0  # 0 = the reference's 256 cap

    def _c(self) -> _Cfg:
        return _Cfg(self.s, self.k, self.t, self.bs, self.workers, self.scale,
                    self.selector_threshold, self.seed, self.smp_fraction,
                    self.pub_model_path.encode() if self.pub_model_path else None,
                    self.device, self.max_workers)


@dataclass
class PipelineStats:
    workers: List[WorkerStats] = field(default_factory=list)
    timing: Optional[Timing] = None


def chunk_count(raw: bytes, cfg: CompressConfig = CompressConfig()) -> int:
    """Chunks compress() writes for this input (host-only plan, pipeline.cpp:32-52)."""
    c = cfg._c()
    n = C.c_size_t()
    _check(lib().pmklc_chunk_count(raw, C.c_size_t(len(raw)), C.byref(c), C.byref(n)))
    return n.value


def compress(raw: bytes, cfg: CompressConfig = CompressConfig(),
             stats: Optional[PipelineStats] = None) -> bytes:
    """pmklc::compress — returns the PMKL container (byte-identical to the reference)."""
    c = cfg._c()
    out = C.POINTER(C.c_uint8)()
    n = C.c_size_t()
    cap = chunk_count(raw, cfg) if stats is not None else 0
    st = (Stats * max(cap, 1))() if stats is not None else None
    nch = C.c_size_t()
    tm = Timing()
    _check(lib().pmklc_compress(raw, C.c_size_t(len(raw)), C.byref(c), C.byref(out), C.byref(n),
                                st, C.c_size_t(cap), C.byref(nch), C.byref(tm)))
    if stats is not None:
        stats.workers = _worker_stats(st, min(nch.value, cap))
        stats.timing = tm
    return _take(out, n.value)


def compress_file(in_path: str, out_path: str, cfg: CompressConfig = CompressConfig(),
                  block_bytes: int = 0, timing: Optional[Timing] = None) -> None:
    """File to file with bounded host memory: the input streams into HBM block
    by block (pinned double buffer, read overlapping copy); same container."""
    c = cfg._c()
    tm = timing if timing is not None else Timing()
    _check(lib().pmklc_compress_file(in_path.encode(), out_path.encode(), C.byref(c),
                                     C.c_size_t(block_bytes), C.byref(tm)))


def decompress_file(in_path: str, out_path: str, pub_model_path: str = "", device: int = 0,
                    block_bytes: int = 0, timing: Optional[Timing] = None) -> None:
    """Container file to original file, the output streamed out of HBM block by block."""
    tm = timing if timing is not None else Timing()
    _check(lib().pmklc_decompress_file(in_path.encode(), out_path.encode(),
                                       pub_model_path.encode() if pub_model_path else None, device,
                                       C.c_size_t(block_bytes), C.byref(tm)))


def compress_device(d_ptr: int, n: int, cfg: CompressConfig = CompressConfig(),
                    timing: Optional[Timing] = None) -> bytes:
    """compress with the input already in device memory (pointer as int)."""
    c = cfg._c()
    out = C.POINTER(C.c_uint8)()
    on = C.c_size_t()
    tm = timing if timing is not None else Timing()
    _check(lib().pmklc_compress_device(C.c_void_p(d_ptr), C.c_size_t(n), C.byref(c), C.byref(out),
                                       C.byref(on), None, C.c_size_t(0), None, C.byref(tm)))
    return _take(out, on.value)


def decompress(container: bytes, pub_model_path: str = "", workers: int = 1,
               stats: Optional[PipelineStats] = None, device: int = 0) -> bytes:
    """pmklc::decompress — bit-exact inverse of compress."""
    out = C.POINTER(C.c_uint8)()
    n = C.c_size_t()
    cap = 0
    if stats is not None:  # chunk count from the container header (container.cpp:53)
        cn = C.c_size_t()
        if lib().pmklc_container_chunks(container, C.c_size_t(len(container)), C.byref(cn)) == 0:
            cap = cn.value
    st = (Stats * max(cap, 1))() if stats is not None else None
    tm = Timing()
    _check(lib().pmklc_decompress(container, C.c_size_t(len(container)),
                                  pub_model_path.encode() if pub_model_path else None, workers,
                                  device, C.byref(out), C.byref(n), st, C.c_size_t(cap),
                                  C.byref(tm)))
    if stats is not None:
        stats.workers = _worker_stats(st, cap)
        stats.timing = tm
    return _take(out, n.value)


def decompress_to_device(container: bytes, pub_model_path: str = "", device: int = 0,
                         timing: Optional[Timing] = None):
    """Returns (device_ptr:int, length); free with device_free."""
    d = C.c_void_p()
    n = C.c_size_t()
    tm = timing if timing is not None else Timing()
    _check(lib().pmklc_decompress_to_device(container, C.c_size_t(len(container)),
                                            pub_model_path.encode() if pub_model_path else None,
                                            device, C.byref(d), C.byref(n), C.byref(tm)))
    return d.value, n.value


def device_free(ptr: int) -> None:
    lib().pmklc_device_free(C.c_void_p(ptr))


def encode_chunks(tokens, chunk_lens: Sequence[int], inbound: Sequence[bytes], flags: int, k: int,
                  t: int, bs: int, scale: int, dm_seed: int, pub_model_path: str = "",
                  device: int = 0, priv_model: bytes = b"") -> List[bytes]:
    """Batched pmklc::encode_chunk_standalone (ChunkCodeSpec, pipeline.hpp:69-78):
    flags & 1 uses the public model file, flags & 2 the private model given as
    its PMKW bytes (the container's SPrM blob)."""
    import numpy as np
    tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
    nc = len(chunk_lens)
    lens = (C.c_uint64 * nc)(*chunk_lens)
    ib = (C.c_char_p * nc)(*[bytes(b) for b in inbound])
    ibl = (C.c_size_t * nc)(*[len(b) for b in inbound])
    pays = (C.POINTER(C.c_uint8) * nc)()
    pl = (C.c_size_t * nc)()
    _check(lib().pmklc_encode_chunks(tokens.ctypes.data_as(C.c_void_p), lens, C.c_size_t(nc),
                                     C.cast(ib, C.c_void_p), ibl, flags,
                                     pub_model_path.encode() if pub_model_path else None,
                                     priv_model or None, C.c_size_t(len(priv_model)), k, t, bs,
                                     scale, C.c_uint64(dm_seed), device, pays, pl))
    return [_take(pays[i], pl[i]) for i in range(nc)]


def dump_chunk(tokens, flags: int, k: int, t: int, bs: int, scale: int, dm_seed: int,
               pub_model_path: str = "", inbound: bytes = b"", max_steps: int = 0, device: int = 0):
    """One chunk with its first max_steps mixed-probability tables: (payload, probs)."""
    import numpy as np
    tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
    V = 1 << (2 * k)
    probs = np.zeros((max(max_steps, 1), bs, V), dtype=np.float32)
    out = C.POINTER(C.c_uint8)()
    n = C.c_size_t()
    _check(lib().pmklc_dump_chunk(tokens.ctypes.data_as(C.c_void_p), C.c_uint64(len(tokens)), flags,
                                  pub_model_path.encode() if pub_model_path else None, k, t, bs,
                                  scale, C.c_uint64(dm_seed), inbound, C.c_size_t(len(inbound)),
                                  device, probs.ctypes.data_as(C.c_void_p), C.c_uint64(max_steps),
                                  C.byref(out), C.byref(n)))
    return _take(out, n.value), probs[:max_steps]


def quantize(probs, device: int = 0):
    """pmklc::quantize on the device for a [rows, width] float32 array -> uint32 freqs."""
    import numpy as np
    p = np.ascontiguousarray(np.atleast_2d(probs), dtype=np.float32)
    f = np.zeros(p.shape, dtype=np.uint32)
    _check(lib().pmklc_quantize(p.ctypes.data_as(C.c_void_p), C.c_uint64(p.shape[0]),
                                p.shape[1], device, f.ctypes.data_as(C.c_void_p)))
    return f


def skmer_encode(codes: bytes, s: int, k: int, device: int = 0):
    """pmklc::encode on base codes 0..3 -> numpy uint32 tokens."""
    import numpy as np
    n = len(codes)
    mcap = (n - k) // s + 1 if n >= k else 0
    tok = np.zeros(max(mcap, 1), dtype=np.uint32)
    m = C.c_uint64()
    _check(lib().pmklc_skmer_encode(codes, C.c_uint64(n), s, k, device,
                                    tok.ctypes.data_as(C.c_void_p), C.byref(m)))
    return tok[: m.value]


def skmer_encode_packed_device(d_packed: int, n_bases: int, s: int, k: int, d_tokens: int,
                               stream: int = 0, u16: bool = False) -> None:
    """Device tokenizer; u16=True writes 2-byte tokens (k <= 8)."""
    f = lib().pmklc_skmer_encode_packed_device_u16 if u16 else lib().pmklc_skmer_encode_packed_device
    _check(f(C.c_void_p(d_packed), C.c_uint64(n_bases), s, k, C.c_void_p(d_tokens),
             C.c_void_p(stream)))


def plan_chunks(m: int, workers: int, bs: int, t: int, smp_per_myriad: int):
    """pmklc::plan_chunks (host logic): (starts, lens, bs, snapshot_steps)."""
    cap = max(workers, 1)
    st = (C.c_uint64 * cap)()
    ln = (C.c_uint64 * cap)()
    sn = (C.c_uint64 * cap)()
    cnt = C.c_size_t()
    bso = C.c_uint32()
    _check(lib().pmklc_plan_chunks(C.c_uint64(m), workers, bs, t, C.c_uint16(smp_per_myriad), st, ln,
                                   sn, C.c_size_t(cap), C.byref(cnt), C.byref(bso)))
    n = cnt.value
    return list(st[:n]), list(ln[:n]), bso.value, list(sn[:n])


def schedule(lens: Sequence[int], bs: int, t: int, smp_per_myriad: int):
    """Tick schedule of Step-wise Model Passing (host logic): per chunk
    (offset, src, src_steps, model_steps) and the tick count."""
    nc = len(lens)
    L = (C.c_uint64 * nc)(*lens)
    off = (C.c_int64 * nc)()
    src = (C.c_int64 * nc)()
    ss = (C.c_uint64 * nc)()
    ms = (C.c_uint64 * nc)()
    ticks = C.c_int64()
    _check(lib().pmklc_schedule(L, C.c_size_t(nc), bs, t, C.c_uint16(smp_per_myriad), off, src, ss,
                                ms, C.byref(ticks)))
    return list(off), list(src), list(ss), list(ms), ticks.value


def schedule_slots(lens: Sequence[int], bs: int, t: int, smp_per_myriad: int, rank: int = 0,
                   world: int = 1):
    """State/tape slot per chunk (-1: never steps / other rank) and the slot count."""
    nc = len(lens)
    L = (C.c_uint64 * max(nc, 1))(*lens)
    sl = (C.c_int32 * max(nc, 1))()
    ns = C.c_int32()
    _check(lib().pmklc_schedule_slots(L, C.c_size_t(nc), bs, t, C.c_uint16(smp_per_myriad), rank,
                                      world, sl, C.byref(ns)))
    return list(sl[:nc]), ns.value


def synth(kind: str, n: int, seed: int, extra: int = 0) -> bytes:
    """Seeded synthetic DNA: markov3 | uniform | genome | species | packed."""
    buf = (C.c_uint8 * max(n, 1))()
    L = lib()
    if kind == "markov3":
        L.pmklc_synth_markov3(buf, C.c_uint64(n), C.c_uint64(seed))
    elif kind == "uniform":
        L.pmklc_synth_uniform(buf, C.c_uint64(n), C.c_uint64(seed))
    elif kind == "genome":
        L.pmklc_synth_genome(buf, C.c_uint64(n), C.c_uint64(seed), C.c_uint32(extra or 10))
    elif kind == "species":
        L.pmklc_synth_species(buf, C.c_uint64(n), C.c_uint64(seed), C.c_uint64(extra))
    elif kind == "packed":
        L.pmklc_synth_packed_codes(buf, C.c_uint64(n), C.c_uint64(seed))
    else:
        raise ValueError(kind)
    return bytes(buf)[:n]


def pretrain_public(corpus: Sequence[bytes], s: int = 3, k: int = 3, t: int = 32, batch: int = 64,
                    scale: int = 4, epochs: int = 2, seed: int = 0, device: int = 0,
                    timing: Optional[list] = None) -> bytes:
    """pmklc::pretrain_public (training.cpp:43-60, TrainConfig defaults): the
    trained 2-layer public model (SPuM) as PMKW bytes, byte-identical to the
    reference's serialize_model of its result."""
    n = len(corpus)
    files = (C.c_char_p * max(n, 1))(*[bytes(f) for f in corpus])
    lens = (C.c_size_t * max(n, 1))(*[len(f) for f in corpus])
    out = C.POINTER(C.c_uint8)()
    on = C.c_size_t()
    ms = C.c_double()
    _check(lib().pmklc_pretrain_public(C.cast(files, C.c_void_p), lens, C.c_size_t(n), s, k, t, batch,
                                       scale, epochs, C.c_uint64(seed), device, C.byref(out),
                                       C.byref(on), C.byref(ms)))
    if timing is not None:
        timing.append(ms.value)
    return _take(out, on.value)


def write_bigru(path: str, k: int, t: int, scale: int, seed: int, layers: int = 2) -> int:
    """Write a seeded (untrained) BiGRU model file (PMKW); returns its FNV-1a fingerprint."""
    fp = C.c_uint64()
    _check(lib().pmklc_write_bigru(path.encode(), k, t, scale, layers, C.c_uint64(seed), C.byref(fp)))
    return fp.value


def bench_kernel(name: str, chunks: int, scale: int = 4, rows: int = 320, t: int = 32,
                 iters: int = 20, device: int = 0):
    """Live microbenchmark: (avg_ms per launch, flops per launch, bytes per launch)."""
    ms, fl, by = C.c_double(), C.c_double(), C.c_double()
    _check(lib().pmklc_bench_kernel(name.encode(), device, chunks, scale, rows, t, iters,
                                    C.byref(ms), C.byref(fl), C.byref(by)))
    return ms.value, fl.value, by.value


def dist_plan(lens: Sequence[int], bs: int, t: int, smp_per_myriad: int, rank: int, world: int):
    """This rank's cross-rank SMP handoffs [(tick, src, dst, peer, send)] and its
    number of model steps (host logic of PMKLC-M, no GPU needed)."""
    nc = len(lens)
    L = (C.c_uint64 * nc)(*lens)
    cap = 4 * nc + 4
    tk = (C.c_int64 * cap)()
    sr, ds, pe = (C.c_int32 * cap)(), (C.c_int32 * cap)(), (C.c_int32 * cap)()
    se = (C.c_uint8 * cap)()
    nops, steps = C.c_size_t(), C.c_uint64()
    _check(lib().pmklc_dist_plan(L, C.c_size_t(nc), bs, t, C.c_uint16(smp_per_myriad), rank, world,
                                 tk, sr, ds, pe, se, C.c_size_t(cap), C.byref(nops), C.byref(steps)))
    return [(tk[i], sr[i], ds[i], pe[i], bool(se[i])) for i in range(nops.value)], steps.value


class DistContext:
    """PMKLC-M communicator for this process's GPU. Uses torch.distributed
    (any backend) only to broadcast the 128-byte NCCL id from rank 0."""

    def __init__(self, rank: int, world: int, device: int):
        import torch.distributed as dist
        buf = (C.c_uint8 * 128)()
        if rank == 0:
            _check(lib().pmklc_nccl_id(buf))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0)
        idb = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _check(lib().pmklc_dist_create(idb, rank, world, device, C.byref(h)))
        self.h, self.rank, self.world, self.device = h, rank, world, device

    def compress(self, raw: bytes, cfg: CompressConfig, timing: Optional[Timing] = None) -> bytes:
        c = cfg._c()
        out = C.POINTER(C.c_uint8)()
        n = C.c_size_t()
        tm = timing if timing is not None else Timing()
        _check(lib().pmklc_compress_dist(self.h, raw, None, C.c_size_t(len(raw)), C.byref(c),
                                         C.byref(out), C.byref(n), C.byref(tm)))
        return _take(out, n.value)

    def compress_device(self, d_ptr: int, n: int, cfg: CompressConfig,
                        timing: Optional[Timing] = None) -> bytes:
        c = cfg._c()
        out = C.POINTER(C.c_uint8)()
        on = C.c_size_t()
        tm = timing if timing is not None else Timing()
        _check(lib().pmklc_compress_dist(self.h, None, C.c_void_p(d_ptr), C.c_size_t(n), C.byref(c),
                                         C.byref(out), C.byref(on), C.byref(tm)))
        return _take(out, on.value)

    def decompress(self, blob: bytes, pub_model_path: str = "",
                   timing: Optional[Timing] = None) -> bytes:
        out = C.POINTER(C.c_uint8)()
        n = C.c_size_t()
        tm = timing if timing is not None else Timing()
        _check(lib().pmklc_decompress_dist(self.h, blob, C.c_size_t(len(blob)),
                                           pub_model_path.encode() if pub_model_path else None,
                                           C.byref(out), C.byref(n), C.byref(tm)))
        return _take(out, n.value)

    def decompress_to_device(self, blob: bytes, pub_model_path: str = "",
                             timing: Optional[Timing] = None):
        """(device_ptr, length) on rank 0 ((0, 0) elsewhere); free with device_free."""
        d = C.c_void_p()
        n = C.c_size_t()
        tm = timing if timing is not None else Timing()
        _check(lib().pmklc_decompress_dist_to_device(
            self.h, blob, C.c_size_t(len(blob)),
            pub_model_path.encode() if pub_model_path else None, C.byref(d), C.byref(n),
            C.byref(tm)))
        return d.value or 0, n.value

    def close(self):
        if self.h:
            lib().pmklc_dist_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------- metrics
def compression_ratio(compressed_bytes: int, source_bytes: int) -> float:
    """Eq. 3, bits per base (bench.cpp:15-18); PmklcError EmptySource for 0."""
    out = C.c_double()
    _check(lib().pmklc_compression_ratio(C.c_uint64(compressed_bytes), C.c_uint64(source_bytes),
                                         C.byref(out)))
    return out.value


def throughput(source_bytes: int, ct_s: float, dt_s: float) -> float:
    """Eq. 4, bytes/s over CT + DT (bench.cpp:20-24); PmklcError ZeroTime."""
    out = C.c_double()
    _check(lib().pmklc_throughput(C.c_uint64(source_bytes), C.c_double(ct_s), C.c_double(dt_s),
                                  C.byref(out)))
    return out.value


def robustness(crs: Sequence[float]) -> float:
    """Eq. 5, CRP in percent with the n-1 denominator (bench.cpp:26-36)."""
    n = len(crs)
    arr = (C.c_double * max(n, 1))(*crs)
    out = C.c_double()
    _check(lib().pmklc_robustness(arr, C.c_size_t(n), C.byref(out)))
    return out.value


def block_ratios(container: bytes) -> List[float]:
    """Per data block compression ratios of a container (the CRP population)."""
    cn = C.c_size_t()
    _check(lib().pmklc_container_chunks(container, C.c_size_t(len(container)), C.byref(cn)))
    arr = (C.c_double * max(cn.value, 1))()
    cnt = C.c_size_t()
    _check(lib().pmklc_block_ratios(container, C.c_size_t(len(container)), arr,
                                    C.c_size_t(cn.value), C.byref(cnt)))
    return list(arr[: min(cnt.value, cn.value)])


class DatasetResult(C.Structure):
    """DatasetResult (bench.hpp:22-29)."""
    _fields_ = [("_name", C.c_char * 256), ("source_bytes", C.c_uint64),
                ("compressed_bytes", C.c_uint64), ("ct_s", C.c_double), ("dt_s", C.c_double),
                ("cr", C.c_double), ("thp", C.c_double), ("_verified", C.c_int32)]

    @property
    def name(self) -> str:
        return self._name.decode()

    @property
    def verified(self) -> bool:
        return bool(self._verified)


class MetricsReport(C.Structure):
    """MetricsReport (bench.hpp:31-36) + the device HBM peak."""
    _fields_ = [("mean_cr", C.c_double), ("crp_percent", C.c_double),
                ("peak_mem_bytes", C.c_uint64), ("peak_device_bytes", C.c_uint64)]


def run_benchmark(paths: Sequence[str], cfg: CompressConfig = CompressConfig(), csv_path: str = "",
                  fault_flip_mid: bool = False):
    """run_benchmark (bench.cpp:67-114): (rows, report)."""
    n = len(paths)
    ps = (C.c_char_p * max(n, 1))(*[p.encode() for p in paths])
    rows = (DatasetResult * max(n, 1))()
    rep = MetricsReport()
    c = cfg._c()
    _check(lib().pmklc_run_benchmark(ps, C.c_size_t(n), C.byref(c),
                                     csv_path.encode() if csv_path else None,
                                     1 if fault_flip_mid else 0, rows, C.byref(rep)))
    return list(rows[:n]), rep


def fnv1a64(b: bytes) -> int:
    """FNV-1a-64 (bytes.hpp:17-24)."""
    f = lib().pmklc_fnv1a64
    f.restype = C.c_uint64
    return int(f(b, C.c_size_t(len(b))))


def device_equal(d_ptr: int, d_ref_ptr: int, n: int, device: int = 0) -> bool:
    """True when n bytes at device pointer d_ptr equal those at d_ref_ptr
    (verification of device-resident decompression output; torch compares)."""
    import torch
    cuda = C.CDLL("libcuda.so.1")
    a = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    b = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    torch.cuda.synchronize(device)
    for dst, src in ((a, d_ptr), (b, d_ref_ptr)):
        if cuda.cuMemcpyDtoD_v2(C.c_uint64(dst.data_ptr()), C.c_uint64(src), C.c_size_t(n)) != 0:
            raise PmklcError(101, "cuMemcpyDtoD failed")
    torch.cuda.synchronize(device)
    return bool(torch.equal(a, b))


def version() -> str:
    return lib().pmklc_version().decode()
