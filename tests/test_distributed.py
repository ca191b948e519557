"""CPU, world_size 2 over gloo: the PMKLC-M multi-rank path's host logic.

Each rank takes its chunks and its cross-rank SMP handoffs from the
product's plan (`pmklc_dist_plan`: chunk c on rank c % world, a handoff whose
source and destination live on different ranks becomes a send/recv at the
handoff tick). The compute of a chunk is done by the oracle port (the checker;
the GPU engine runs the same plan with NCCL send/recv of the device state
slot), snapshots travel over gloo exactly where the plan says, and rank 0
checks every chunk's codestream against the single-process reference
container. This pins the routing (who sends which state to whom, when, in
which order) that the NCCL path executes.
"""
import os
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracles as O

CASES = [
    # (n bytes, seed, cfg) -- SMP chains with snapshots after training starts,
    # inherited sources (snapshot during warm-up) and SMP off
    (60000, 31, dict(t=8, bs=32, scale=16, workers=5, smp=0.3)),
    (40000, 32, dict(t=8, bs=16, scale=16, workers=4, smp=0.05)),
    (40000, 33, dict(t=8, bs=16, scale=16, workers=3, smp=0.0)),
]


def container_payloads(blob):
    W = struct.unpack_from("<I", blob, 48)[0]
    out = []
    for i in range(W):
        e = 52 + 36 * i
        _, _, off, plen = struct.unpack_from("<QQQQ", blob, e)
        out.append(blob[off:off + plen])
    return out


def run_rank(rank, world, port_path, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = "29533"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes as C
    import paper_2507_12805_b200 as P
    port = O.port()
    results = []
    for n, seed, kw in CASES:
        raw = P.synth("markov3", n, seed)
        a = np.frombuffer(raw, np.uint8)
        codes = (((a >> 1) ^ (a >> 2)) & 3).astype(np.uint8).tobytes()
        tok, _ = port.skmer_encode(codes, 3, 3)
        myriad = int(round(kw["smp"] * 10000))
        starts, lens, bs, snaps = P.plan_chunks(len(tok), kw["workers"], kw["bs"], kw["t"], myriad)
        W = len(lens)
        ops, steps = P.dist_plan(lens, bs, kw["t"], myriad, rank, world)
        off, src, src_steps, msteps, ticks = P.schedule(lens, bs, kw["t"], myriad)
        # exchange op lists: every send must meet the matching recv on the peer
        all_ops = [None] * world
        dist.all_gather_object(all_ops, ops)
        for r in range(world):
            for (tk, s, d, peer, send) in all_ops[r]:
                assert (tk, s, d, r, not send) in all_ops[peer]
        # run my chunks in ascending order; the dm seed is the master seed's first draw
        dm_seed = struct.unpack_from("<Q", port.compress(b"", O.make_cfg(**kw)), 16)[0]
        mine = [c for c in range(W) if c % world == rank]
        snapshots = {}  # chunk -> snapshot bytes at its emit step
        payloads = {}
        sends_by_src = {}
        for (tk, s, d, peer, send) in ops:
            if send:
                sends_by_src.setdefault(s, []).append((d, peer))
        for c in mine:
            L = lens[c] // bs
            used = L * bs
            t0 = starts[c]
            ctoks = np.ascontiguousarray(tok[t0:t0 + used], dtype=np.uint32)
            inbound = b""
            if src[c] >= 0:
                if src[c] % world == rank:
                    inbound = snapshots[src[c]]
                else:
                    sz = torch.zeros(1, dtype=torch.int64)
                    dist.recv(sz, src=src[c] % world, tag=2 * c)
                    buf = torch.zeros(int(sz.item()), dtype=torch.uint8)
                    dist.recv(buf, src=src[c] % world, tag=2 * c + 1)
                    inbound = bytes(buf.numpy())
            # state this chunk hands on: after src_steps of the dependants
            snap_at = 0
            dep = [d for d in range(W) if src[d] == c]
            if dep:
                snap_at = src_steps[dep[0]] + kw["t"]
            pay = C.POINTER(C.c_uint8)()
            pn = C.c_size_t()
            sn = C.POINTER(C.c_uint8)()
            snn = C.c_size_t()
            rc = port.lib.orc_encode_chunk_snap(
                ctoks.ctypes.data_as(C.c_void_p), C.c_uint64(len(ctoks)), 4, None, 3, kw["t"], bs,
                kw["scale"], C.c_uint64(dm_seed), inbound, C.c_size_t(len(inbound)),
                C.c_uint64(snap_at), C.byref(pay), C.byref(pn), C.byref(sn), C.byref(snn))
            assert rc == 0, port.lib.orc_last_error()
            payloads[c] = C.string_at(pay, pn.value)
            snapshots[c] = C.string_at(sn, snn.value) if snn.value else b""
            for d, peer in sends_by_src.get(c, []):
                b = torch.frombuffer(bytearray(snapshots[c]), dtype=torch.uint8)
                dist.send(torch.tensor([b.numel()], dtype=torch.int64), dst=peer, tag=2 * d)
                dist.send(b, dst=peer, tag=2 * d + 1)
        gathered = [None] * world
        dist.all_gather_object(gathered, payloads)
        if rank == 0:
            merged = {}
            for g in gathered:
                merged.update(g)
            want = container_payloads(O.ref().compress(raw, O.make_cfg(**kw))
                                      if O.REF_SO.exists() else port.compress(raw, O.make_cfg(**kw)))
            results.append(all(merged[c] == want[c] for c in range(W)) and len(merged) == W)
    if rank == 0:
        q.put(results)
    dist.barrier()
    dist.destroy_process_group()


def test_pmklc_m_routing_world2_gloo(port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=run_rank, args=(r, 2, str(O.PORT_SO), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert res == [True] * len(CASES)


def test_dist_plan_partitions_work(P):
    lens = [16 * 100] * 7
    total = 0
    for world in (1, 2, 3, 4):
        steps = []
        for r in range(world):
            ops, st = P.dist_plan(lens, 16, 8, 2000, r, world)
            steps.append(st)
            for (tk, s, d, peer, send) in ops:
                assert (s % world == r) == send and (d % world == r) != send
        assert sum(steps) == 7 * 92
