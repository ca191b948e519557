"""ctypes access to the two CPU checkers (TEST INFRASTRUCTURE).

* ``REF``  — oracle/_ref/libpmklc_ref.so: the unmodified reference core compiled
  from /root/reference/proj/core/src by oracle/Makefile, behind ref_shim.cpp.
* ``PORT`` — oracle/_ref/liboracle.so: the C restatement oracle/pmklc_oracle.c.

Both export the same entry points (``pmref_*`` / ``orc_*``), wrapped here by
``Checker`` so a test can run one case through either. Only tests/, smoke()
and bench.py's cpu_baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libpmklc_ref.so"
PORT_SO = ROOT / "oracle" / "_ref" / "liboracle.so"

ERRC = [
    "LengthMismatch", "TokenOutOfRange", "NotOverlapping", "ShapeMismatch", "StaleTape",
    "ContextLengthMismatch", "ChecksumMismatch", "ArchitectureMismatch", "MissingLogits",
    "BatchMismatch", "InvalidDistribution", "StreamExhausted", "BadMagic", "UnsupportedVersion",
    "TableInconsistent", "ConfigInvalid", "IoError", "SpumMissing", "CorruptStream", "CorpusEmpty",
    "TargetTooShort", "EmptySource", "ZeroTime", "EmptyList", "VerificationFailed",
]


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.errc = ERRC[code - 1] if 1 <= code <= len(ERRC) else "Unknown"
        super().__init__(f"{self.errc}: {msg}")


class Cfg(C.Structure):
    _fields_ = [("s", C.c_uint32), ("k", C.c_uint32), ("t", C.c_uint32), ("bs", C.c_uint32),
                ("workers", C.c_uint32), ("scale", C.c_uint32), ("threshold", C.c_uint64),
                ("seed", C.c_uint64), ("smp", C.c_float), ("pub_path", C.c_char_p)]


class ChunkStats(C.Structure):
    _fields_ = [("tokens", C.c_uint64), ("uniform_coded", C.c_uint64), ("pub_calls", C.c_uint64),
                ("priv_calls", C.c_uint64), ("dyn_calls", C.c_uint64),
                ("snapshot_recv_hash", C.c_uint64), ("snapshot_sent_hash", C.c_uint64),
                ("early_loss_bits", C.c_double)]


def make_cfg(s=3, k=3, t=32, bs=320, workers=1, scale=4, threshold=500_000_000, seed=42,
             smp=0.05, pub_path=None) -> Cfg:
    return Cfg(s, k, t, bs, workers, scale, threshold, seed, smp,
               pub_path.encode() if pub_path else None)


class Checker:
    def __init__(self, so: Path, prefix: str):
        if not so.exists():
            raise FileNotFoundError(f"{so} missing: run `make -C oracle` (build())")
        self.lib = C.CDLL(str(so))
        self.p = prefix
        getattr(self.lib, prefix + "last_error").restype = C.c_char_p

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc != 0:
            raise CheckerError(rc, self._f("last_error")().decode())

    def _take(self, ptr, n) -> bytes:
        b = C.string_at(ptr, n)
        self._f("free")(ptr)
        return b

    def compress(self, raw: bytes, cfg: Cfg, with_stats=False):
        out = C.POINTER(C.c_uint8)()
        n = C.c_size_t()
        cap = 4096
        st = (ChunkStats * cap)() if with_stats else None
        nch = C.c_size_t()
        self._check(self._f("compress")(raw, C.c_size_t(len(raw)), C.byref(cfg), C.byref(out), C.byref(n),
                                        st, C.c_size_t(cap if with_stats else 0), C.byref(nch)))
        data = self._take(out, n.value)
        if with_stats:
            return data, [st[i] for i in range(nch.value)]
        return data

    def decompress(self, blob: bytes, pub_path=None, workers=1, with_stats=False):
        out = C.POINTER(C.c_uint8)()
        n = C.c_size_t()
        cap = 4096
        st = (ChunkStats * cap)() if with_stats else None
        self._check(self._f("decompress")(blob, C.c_size_t(len(blob)), pub_path.encode() if pub_path else None,
                                          workers, C.byref(out), C.byref(n), st,
                                          C.c_size_t(cap if with_stats else 0)))
        data = self._take(out, n.value)
        if with_stats:
            return data, st
        return data

    def skmer_encode(self, codes: bytes, s: int, k: int, workers: int = 1):
        import numpy as np
        n = len(codes)
        m_cap = (n - k) // s + 1 if n >= k else 0
        tok = np.zeros(max(m_cap, 1), dtype=np.uint32)
        res = np.zeros(max(n, 1), dtype=np.uint8)
        m = C.c_uint64()
        rn = C.c_uint64()
        self._check(self._f("skmer_encode")(codes, C.c_uint64(n), s, k, workers,
                                            tok.ctypes.data_as(C.c_void_p), C.byref(m),
                                            res.ctypes.data_as(C.c_void_p), C.byref(rn)))
        return tok[: m.value].copy(), bytes(res[: rn.value])

    def quantize(self, p):
        import numpy as np
        p = np.ascontiguousarray(p, dtype=np.float32)
        f = np.zeros(len(p), dtype=np.uint32)
        self._check(self._f("quantize")(p.ctypes.data_as(C.c_void_p), len(p),
                                        f.ctypes.data_as(C.c_void_p)))
        return f

    def uniform_dist(self, n):
        import numpy as np
        f = np.zeros(n, dtype=np.uint32)
        self._check(self._f("uniform_dist")(n, f.ctypes.data_as(C.c_void_p)))
        return f

    def range_encode(self, freqs, dist_of, syms) -> bytes:
        import numpy as np
        freqs = np.ascontiguousarray(freqs, dtype=np.uint32)
        dist_of = np.ascontiguousarray(dist_of, dtype=np.uint32)
        syms = np.ascontiguousarray(syms, dtype=np.uint32)
        out = C.POINTER(C.c_uint8)()
        n = C.c_size_t()
        self._check(self._f("range_encode")(freqs.ctypes.data_as(C.c_void_p), freqs.shape[1],
                                            dist_of.ctypes.data_as(C.c_void_p),
                                            syms.ctypes.data_as(C.c_void_p), C.c_size_t(len(syms)),
                                            C.byref(out), C.byref(n)))
        return self._take(out, n.value)

    def det(self, which: int, x):
        import numpy as np
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.zeros_like(x)
        self._check(self._f("det")(which, x.ctypes.data_as(C.c_void_p),
                                   y.ctypes.data_as(C.c_void_p), C.c_size_t(len(x))))
        return y

    def softmax(self, x):
        import numpy as np
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.zeros_like(x)
        self._check(self._f("softmax")(x.ctypes.data_as(C.c_void_p),
                                       y.ctypes.data_as(C.c_void_p), C.c_size_t(len(x))))
        return y

    def bigru_predict(self, path: str, ctx, vocab: int):
        import numpy as np
        ctx = np.ascontiguousarray(ctx, dtype=np.uint32)
        rows, steps = ctx.shape
        out = np.zeros((rows, vocab), dtype=np.float32)
        self._check(self._f("bigru_predict")(path.encode(), ctx.ctypes.data_as(C.c_void_p),
                                             C.c_int64(rows), C.c_int64(steps),
                                             out.ctypes.data_as(C.c_void_p)))
        return out

    def dump_chunk(self, tokens, flags, k, t, bs, scale, dm_seed, pub_path=None, inbound=b"",
                   max_steps=0):
        """Replay one chunk; returns (payload, snapshot, probs[steps, bs, V])."""
        import numpy as np
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        V = 1 << (2 * k)
        probs = np.zeros((max(max_steps, 1), bs, V), dtype=np.float32)
        pay = C.POINTER(C.c_uint8)()
        pn = C.c_size_t()
        sn = C.POINTER(C.c_uint8)()
        snn = C.c_size_t()
        self._check(self._f("dump_chunk")(
            tokens.ctypes.data_as(C.c_void_p), C.c_uint64(len(tokens)), flags,
            pub_path.encode() if pub_path else None, k, t, bs, scale, C.c_uint64(dm_seed),
            inbound, C.c_size_t(len(inbound)), probs.ctypes.data_as(C.c_void_p), C.c_uint64(max_steps),
            C.byref(pay), C.byref(pn), C.byref(sn), C.byref(snn)))
        return self._take(pay, pn.value), self._take(sn, snn.value), probs[:max_steps]

    def pretrain_private(self, tokens, k, t, batch, scale, seed, pub_path=None) -> bytes:
        import numpy as np
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        out = C.POINTER(C.c_uint8)()
        n = C.c_size_t()
        self._check(self._f("pretrain_private")(
            tokens.ctypes.data_as(C.c_void_p), C.c_uint64(len(tokens)),
            pub_path.encode() if pub_path else None, k, t, batch, scale, C.c_uint64(seed),
            C.byref(out), C.byref(n)))
        return self._take(out, n.value)


    def fnv(self, b: bytes) -> int:
        """FNV-1a-64 (bytes.hpp:17-24) of a byte string."""
        f = self._f("fnv1a64")
        f.restype = C.c_uint64
        return int(f(b, C.c_size_t(len(b))))

    def pretrain_public(self, corpus, s=3, k=3, t=32, batch=64, scale=4, epochs=2, seed=0) -> bytes:
        """pmklc::pretrain_public (training.cpp:43-60): PMKW bytes of the trained SPuM."""
        n = len(corpus)
        files = (C.c_char_p * max(n, 1))(*[bytes(f) for f in corpus])
        lens = (C.c_size_t * max(n, 1))(*[len(f) for f in corpus])
        out = C.POINTER(C.c_uint8)()
        on = C.c_size_t()
        self._check(self._f("pretrain_public")(C.cast(files, C.c_void_p), lens, C.c_size_t(n), s, k, t,
                                               batch, scale, epochs, C.c_uint64(seed), C.byref(out),
                                               C.byref(on)))
        return self._take(out, on.value)

    def synth(self, kind: str, n: int, seed: int, extra: int = 0) -> bytes:
        """Seeded benchmark inputs (the generators of host/synth.cpp, built
        into the checker library): markov3 | uniform | genome | species."""
        buf = (C.c_uint8 * max(n, 1))()
        f = self._f("synth_" + kind)
        if kind == "genome":
            f(buf, C.c_uint64(n), C.c_uint64(seed), C.c_uint32(extra or 10))
        elif kind == "species":
            f(buf, C.c_uint64(n), C.c_uint64(seed), C.c_uint64(extra))
        else:
            f(buf, C.c_uint64(n), C.c_uint64(seed))
        return bytes(buf)[:n]

    def replay_chunk(self, tokens, flags, k, t, bs, scale, dm_seed, pub_path=None, priv=b"",
                     inbound=b"", snap_at=0, stop_at=0):
        """ChunkWorker replay (reference classes): (payload, snapshot). The
        snapshot is taken after batch step snap_at (0: after the last step
        run); the run stops after stop_at batch steps (0: all); the payload
        is empty unless the chunk ran to completion."""
        import numpy as np
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        pay = C.POINTER(C.c_uint8)()
        pn = C.c_size_t()
        sn = C.POINTER(C.c_uint8)()
        snn = C.c_size_t()
        self._check(self._f("replay_chunk")(
            tokens.ctypes.data_as(C.c_void_p), C.c_uint64(len(tokens)), flags,
            pub_path.encode() if pub_path else None, priv or None, C.c_size_t(len(priv)), k, t,
            bs, scale, C.c_uint64(dm_seed), inbound or None, C.c_size_t(len(inbound)),
            C.c_uint64(snap_at), C.c_uint64(stop_at), C.byref(pay), C.byref(pn), C.byref(sn),
            C.byref(snn)))
        return self._take(pay, pn.value), self._take(sn, snn.value)

    def encode_chunk_standalone(self, tokens, flags, k, t, bs, scale, dm_seed, pub_path=None,
                                priv=b"", inbound=b"") -> bytes:
        """pmklc::encode_chunk_standalone (pipeline.cpp:298-301), the reference's own hook."""
        import numpy as np
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        out = C.POINTER(C.c_uint8)()
        n = C.c_size_t()
        self._check(self._f("encode_chunk_standalone_priv")(
            tokens.ctypes.data_as(C.c_void_p), C.c_uint64(len(tokens)), flags,
            pub_path.encode() if pub_path else None, priv or None, C.c_size_t(len(priv)), k, t,
            bs, scale, C.c_uint64(dm_seed), inbound or None, C.c_size_t(len(inbound)),
            C.byref(out), C.byref(n)))
        return self._take(out, n.value)


def parse_container(blob: bytes):
    """Header fields and per-chunk (token_start, token_len, payload_off,
    payload_len, trailer_len) of a PMKL container (container.cpp:41-88), plus
    the SPrM blob."""
    import struct
    (magic, ver, flags, s, k, t, bs, myriad, dm_seed, sprm_seed, fp, olen,
     nch) = struct.unpack_from("<4sBBBBHIHQQQQI", blob, 0)
    assert magic == b"PMKL"
    chunks = [struct.unpack_from("<QQQQI", blob, 52 + 36 * i) for i in range(nch)]
    at = 52 + 36 * nch
    plen = struct.unpack_from("<Q", blob, at)[0]
    priv = blob[at + 8: at + 8 + plen]
    return {"flags": flags, "s": s, "k": k, "t": t, "bs": bs, "myriad": myriad,
            "dm_seed": dm_seed, "sprm_seed": sprm_seed, "pub_fingerprint": fp,
            "original_len": olen, "chunks": chunks, "priv": priv}


def ref() -> Checker:
    return Checker(REF_SO, "pmref_")


def port() -> Checker:
    return Checker(PORT_SO, "orc_")


def write_spum(path: str, k: int, t: int, scale: int, seed: int, layers: int = 2) -> int:
    """Seeded untrained SPuM file via the reference (acceptance.cpp:58-69)."""
    lib = ref().lib
    fp = C.c_uint64()
    rc = lib.pmref_write_bigru(1 << (2 * k), t, scale, layers, C.c_uint64(seed), path.encode(),
                               C.byref(fp))
    if rc:
        raise CheckerError(rc, "write_bigru")
    return fp.value


def fnv1a64(b: bytes, h: int = 0xcbf29ce484222325) -> int:
    import numpy as np  # noqa: F401  (kept simple; inputs here are small)
    for x in b:
        h ^= x
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h
