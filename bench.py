"""PMKLC B200 benchmark (driver contract in the task statement).

One step = compress + decompress of the whole workload (the paper's Eq. 4
throughput THP = size / (CT + DT)), device-resident input for
`value`, host buffers through the public API for `e2e`.

Default workload (N=1): BASELINE config 3 — a 100 MB synthetic genome (10
order-k Markov segments, k in 2..5, GC bias varied, 1 % copy-repeats),
PMKLC-S block-partitioned into W=128 data blocks, public (seeded, untrained
SPuM) + dynamic models (the selector never enables private and public
together below the 500 MB threshold, mixer.cpp:9-12), reference defaults
s=k=3, t=32, bs=320, scale 4, SMP 0.05.

--impl reference times the reference C++ library itself (oracle/_ref, built
from /root/reference sources) on the host cores over a bounded sample of the
same workload.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Compress/decompress MB/s at 1/2/4/8 B200; bits/base vs CPU reference"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mb", type=float, default=100.0, help="workload size in 10^6 bytes")
    ap.add_argument("--workers", type=int, default=128, help="data blocks W")
    ap.add_argument("--no-spum", action="store_true", help="no public model")
    ap.add_argument("--no-sprm-branch", action="store_true",
                    help="skip the threshold-lowered SPrM+DM (flags 6) run of config 3")
    ap.add_argument("--skip-cpu", action="store_true", help="skip the cpu_baseline leg")
    return ap.parse_args()


def workload(args, tmpdir):
    import paper_2507_12805_b200 as P
    n = int(args.mb * 1e6)
    raw = P.synth("genome", n, 2025, 10)
    cfg = P.CompressConfig(workers=args.workers)
    spum = ""
    if not args.no_spum:
        spum = str(Path(tmpdir) / "spum_k3_t32_s4.bin")
        P.write_bigru(spum, 3, 32, 4, 0xACE3, layers=2)
        cfg.pub_model_path = spum
    models = "DM only (flags 4)" if args.no_spum else "SPuM(seeded)+DM (flags 5, default selector)"
    desc = (f"config3: {n/1e6:g} MB synthetic genome (10 order-k Markov segments k=2..5 + 1% "
            f"repeats), PMKLC-S W={args.workers} blocks, {models}, "
            f"s=k=3 t=32 bs=320 scale=4 smp=0.05")
    return raw, cfg, spum, desc


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, idx):
        self.idx = idx
        self.p = None
        self.f = None

    def start(self):
        """Start sampling and wait for the first sample: NVML initialisation
        can stall the driver for seconds, so it must happen before warm-up."""
        self.__enter__()
        t0 = time.time()
        while self.p and time.time() - t0 < 15:
            try:
                if open(self.f.name).read().strip():
                    break
            except Exception:
                pass
            time.sleep(0.2)
        return self

    def __enter__(self):
        if self.p:
            return self
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        try:
            lines = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        except Exception:
            return None
        if not lines:
            return None
        sm = [float(l[1]) for l in lines if l[1].strip().replace(".", "").isdigit()]
        mx = [float(l[2]) for l in lines if l[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for l in lines for i in range(4)
                          if len(l) > 5 + i and l[5 + i].strip() == "Active"})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(lines)}


def flush_l2(torch, buf):
    buf.add_(1)  # 256 MiB write > 126 MB L2, between timed steps (not timed)


def cpu_sample(raw, cfg, threads):
    """Bounded sample of the workload for the host-CPU reference: `chunks`
    blocks of `steps` batch steps (32 warm-up + the rest model steps). With the
    private model the reference pre-trains it sequentially over the whole
    sample (~130 ms per 320-token step on one core), so that sample is smaller
    (2 blocks x 48 steps: ~100 pre-pass steps) to keep a step within ~30 s."""
    if cfg.selector_threshold == 0:
        chunks, steps = 2, 48
    else:
        chunks, steps = threads, 64
    n = min(len(raw), chunks * 320 * 3 * steps)
    return raw[:n], chunks, steps


def cpu_reference(raw, cfg, spum, threads, reps, warm):
    """The reference library (oracle/_ref) on host cores over a bounded sample."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles as O
    R = O.ref() if O.REF_SO.exists() else O.port()
    kind = "reference" if O.REF_SO.exists() else "port"
    sample, chunks, steps = cpu_sample(raw, cfg, threads)
    n = len(sample)
    c = O.make_cfg(workers=chunks, pub_path=spum or None, threshold=int(cfg.selector_threshold))
    times = []
    blob = b""
    for i in range(warm + reps):
        t0 = time.perf_counter()
        blob = R.compress(sample, c)
        t1 = time.perf_counter()
        out = R.decompress(blob, pub_path=spum or None, workers=chunks)
        t2 = time.perf_counter()
        assert out == sample
        if i >= warm:
            times.append((t1 - t0, t2 - t1))
    ct = sum(t[0] for t in times) / len(times)
    dt = sum(t[1] for t in times) / len(times)
    flags = blob[5] if len(blob) > 5 else 0
    return {"value": n / 1e6 / (ct + dt), "unit": "MB/s", "cores": chunks, "kind": kind,
            "sample": f"first {n} B of the workload, W={chunks} blocks x {steps} batch steps, "
                      f"container flags {flags}; compress {ct:.2f} s + decompress {dt:.2f} s "
                      f"(one host thread per block; the SPrM pre-pass is sequential)",
            "compress_MBps": n / 1e6 / ct, "decompress_MBps": n / 1e6 / dt,
            "bits_per_base": 8.0 * len(blob) / n,
            "n": n}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    tmp = tempfile.mkdtemp(prefix="pmklc_bench_")

    if args.impl == "reference":
        if rank != 0:
            return
        raw, cfg, spum, desc = workload(args, tmp)
        threads = min(os.cpu_count() or 1, 256, args.workers)
        r = cpu_reference(raw, cfg, spum, threads, args.steps, args.warmup)
        line = {"metric": METRIC, "value": r["value"], "unit": "MB/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1000.0 * (r["n"] / 1e6 / r["value"]) if r["value"] else None,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "impl": "reference",
                "config": {"workload": desc, "parallelism": f"{threads} host threads"},
                "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": r["value"], "unit": "MB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "compress_MBps": r["compress_MBps"], "decompress_MBps": r["decompress_MBps"],
                "bits_per_base_sample": r["bits_per_base"]}
        print(json.dumps(line))
        return

    import torch
    import paper_2507_12805_b200 as P

    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")  # host control plane only
    torch.cuda.set_device(local)
    dev = local
    raw, cfg, spum, desc = workload(args, tmp)
    cfg.device = dev
    n = len(raw)
    d_raw = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(f"cuda:{dev}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    ctx = P.DistContext(rank, world, dev) if world > 1 else None

    def bcast(blob):
        if world == 1:
            return blob
        obj = [blob]
        torch.distributed.broadcast_object_list(obj, src=0)
        return obj[0]

    def run_step(cfg):
        """compress (device-resident input) + decompress; PMKLC-M over all ranks."""
        tm_c, tm_d = P.Timing(), P.Timing()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        if ctx is None:
            blob = P.compress_device(d_raw.data_ptr(), n, cfg, tm_c)
        else:
            blob = ctx.compress_device(d_raw.data_ptr(), n, cfg, tm_c)
        e1.record()
        torch.cuda.synchronize()
        blob = bcast(blob)  # container to every rank (not timed)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e1b = torch.cuda.Event(enable_timing=True)
        e1b.record()
        if ctx is None:
            dptr, dlen = P.decompress_to_device(blob, spum, dev, tm_d)
            e2.record()
            torch.cuda.synchronize()
            P.device_free(dptr)
        else:
            out = ctx.decompress(blob, spum, tm_d)
            e2.record()
            torch.cuda.synchronize()
            if rank == 0:
                assert len(out) == n
        c_ms, d_ms = e0.elapsed_time(e1), e1b.elapsed_time(e2)
        return blob, c_ms, d_ms, tm_c.kernel_launches + tm_d.kernel_launches, (tm_c, tm_d)

    def measure(cfg, warmup, steps):
        # correctness of the measured path: lossless round trip (first warm-up)
        blob, _, _, _, _ = run_step(cfg)
        if ctx is None:
            assert P.decompress(blob, spum, device=dev) == raw, "round trip mismatch"
        else:
            out = ctx.decompress(blob, spum)
            if rank == 0:
                assert out == raw, "round trip mismatch"
        for _ in range(max(warmup - 1, 0)):
            run_step(cfg)
        res = {"ct": 0.0, "dt": 0.0, "launches": 0, "flags": blob[5],
               "hot": {"ms": 0.0, "launches": 0, "units": 0, "flops": 0.0},
               "brk": {"sprm_prepass_ms": 0.0, "compress_ticks_ms": 0.0, "decompress_ticks_ms": 0.0}}
        hot, brk = res["hot"], res["brk"]
        with clk:
            for _ in range(steps):
                flush_l2(torch, flush)
                blob, c_ms, d_ms, l, tms = run_step(cfg)
                brk["sprm_prepass_ms"] += tms[0].sprm_ms / steps
                brk["compress_ticks_ms"] += tms[0].model_ms / steps
                brk["decompress_ticks_ms"] += tms[1].model_ms / steps
                for tm in tms:  # dominant kernel, timed on the device inside the timed region
                    hot["ms"] += tm.hot_ms
                    hot["launches"] += tm.hot_launches
                    hot["units"] += tm.hot_units
                    hot["flops"] += tm.hot_flops_per_unit * tm.hot_units
                if world > 1:  # max over ranks, per phase
                    tt = torch.tensor([c_ms, d_ms], dtype=torch.float64)
                    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
                    c_ms, d_ms = float(tt[0]), float(tt[1])
                res["ct"] += c_ms
                res["dt"] += d_ms
                res["launches"] += l
        res["blob"] = blob
        res["value"] = n * steps / 1e6 / ((res["ct"] + res["dt"]) / 1000.0)
        return res

    clk = Clocks(dev).start()
    main_run = measure(cfg, args.warmup, args.steps)
    ct, dt, launches = main_run["ct"], main_run["dt"], main_run["launches"]
    hot, brk, blob = main_run["hot"], main_run["brk"], main_run["blob"]
    tot_ms = ct + dt
    value = main_run["value"]

    # e2e through the public host API (host buffers, H2D/D2H inside)
    e_times = []
    for _ in range(max(1, args.steps // 2)):
        flush_l2(torch, flush)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if ctx is None:
            b2 = P.compress(raw, cfg)
            back = P.decompress(b2, spum, device=dev)
        else:
            b2 = bcast(ctx.compress(raw, cfg))
            back = ctx.decompress(b2, spum)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([el], dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            el = float(tt[0])
        e_times.append(el)
        if rank == 0:
            assert back == raw
    e2e_val = n / 1e6 / (sum(e_times) / len(e_times))

    # config 3's other selector branch: threshold lowered so the private model
    # is pre-trained on the input inside compress (flags 6, SURVEY §8 config 3;
    # the reference never enables SPuM and SPrM together, mixer.cpp:9-12).
    # One warm-up step (the engine paths are already warm from the main run).
    sprm = None
    if not args.no_sprm_branch:
        cfg6 = dataclasses.replace(cfg, selector_threshold=0)
        sprm = measure(cfg6, 1, args.steps)

    line = None
    if rank == 0:
        # roofline of the dominant kernel. With the public model (the default
        # workload) that is the SPuM layer-1 fused BiGRU recurrence, timed on
        # the device around every launch inside the timed steps (stamp kernels
        # on its own stream; in-situ, so co-running DM kernels are included).
        # Bound: exact non-FMA FP32 issue (no tensor cores in EXACT mode); the
        # peak is a live FP32 microbenchmark (MEASURED_PEAKS.json has no FP32
        # figure).
        p_ms, p_fl, _ = P.bench_kernel("fp32_peak", 1, iters=10, device=dev)
        peak_tf = p_fl / (p_ms / 1000.0) / 1e12
        traffic = None
        tfile = ROOT / "profiles" / "roofline_traffic.json"
        tjson = {}
        if tfile.exists():
            try:
                tjson = json.loads(tfile.read_text())
            except Exception:
                tjson = {}
        if hot["launches"]:
            ach_tf = hot["flops"] / (hot["ms"] / 1000.0) / 1e12
            units_per_launch = hot["units"] / hot["launches"]
            t = tjson.get("k_bigru_rec_fused")
            fma_busy = None
            if t and t.get("units"):  # DRAM bytes per chunk-launch x this run's chunks per launch
                traffic = t["dram_bytes_per_launch"] / t["units"] * units_per_launch
                fma_busy = t.get("fma_pipe_busy_pct")
            # the same kernel alone on the GPU (no co-running DM branch), same stamps
            chunks_iso = max(1, int(round(units_per_launch)))
            i_ms, i_fl, _ = P.bench_kernel("bigru_fused", chunks_iso, iters=10, device=dev)
            iso_tf = i_fl / (i_ms / 1000.0) / 1e12 if i_ms > 0 else None
            roof = {"kernel": "k_bigru_rec_fused (SPuM BiGRU layer 1: input projection + "
                              "recurrence, R=320 rows x 2 dirs x t=32 steps per chunk)",
                    "achieved_isolated": iso_tf,
                    "frac_isolated": iso_tf / peak_tf if iso_tf else None,
                    "isolated": f"bench_kernel('bigru_fused', {chunks_iso} chunks): the kernel "
                                "alone; in situ it shares the SMs with the previous tick's DM "
                                "backward (cross-tick pipeline)",
                    "bound": "fp32", "achieved": ach_tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": ach_tf / peak_tf, "traffic": traffic,
                    "timing": "in-situ %globaltimer stamps around every launch in the timed steps",
                    "avg_launch_ms": hot["ms"] / hot["launches"],
                    "chunks_per_launch": units_per_launch,
                    "flops_per_launch": hot["flops"] / hot["launches"],
                    "flops_per_chunk_launch": hot["flops"] / max(hot["units"], 1),
                    "fma_pipe_busy_pct_ncu": fma_busy,
                    "note": "achieved counts MAC flops only; the FP32 pipe also runs the exact "
                            "det-math epilogue and 2 instructions per exact (non-FMA) MAC pair",
                    "peak_source": "live non-FMA FP32 microbenchmark (MEASURED_PEAKS.json has no "
                                   "FP32 figure); EXACT mode cannot use tensor cores"}
        else:  # DM only: the weight-gradient reduction, microbenchmarked live
            chunks = min(args.workers, 64)
            k_ms, k_fl, k_by = P.bench_kernel("gemm_nt", chunks, iters=10, device=dev)
            ach_tf = k_fl / (k_ms / 1000.0) / 1e12
            roof = {"kernel": f"k_gemm_nt (dWk|dbk + dWv|dbv over R*t=10240 rows, {chunks} chunks)",
                    "bound": "fp32", "achieved": ach_tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": ach_tf / peak_tf, "traffic": tjson.get("gemm_nt_dram_bytes_per_launch"),
                    "avg_launch_ms": k_ms, "flops_per_launch": k_fl,
                    "peak_source": "live non-FMA FP32 microbenchmark"}
        cpu = cpu6 = None
        if not args.skip_cpu and world == 1:
            threads = min(os.cpu_count() or 1, 256, args.workers)
            def cpu_leg(c):
                try:
                    full = cpu_reference(raw, c, spum, threads, 1, 0)
                    return {k: full[k] for k in ("value", "unit", "cores", "kind", "sample")}
                except Exception as e:  # report, do not hide
                    return {"value": None, "unit": "MB/s", "cores": threads, "kind": "reference",
                            "sample": f"failed: {e}"}
            cpu = cpu_leg(cfg)
            if sprm is not None:
                cpu6 = cpu_leg(dataclasses.replace(cfg, selector_threshold=0))
        sprm_line = None
        if sprm is not None:
            sprm_line = {
                "workload": desc.replace("SPuM(seeded)+DM (flags 5, default selector)",
                                         "SPrM(pre-trained on the input inside compress)+DM "
                                         "(flags 6, selector_threshold=0)"),
                "container_flags": sprm["flags"], "value": sprm["value"], "unit": "MB/s",
                "warmup": 1, "steps": args.steps,
                "ms_per_step": (sprm["ct"] + sprm["dt"]) / args.steps,
                "compress_MBps": n * args.steps / 1e6 / (sprm["ct"] / 1000.0),
                "decompress_MBps": n * args.steps / 1e6 / (sprm["dt"] / 1000.0),
                "bits_per_base": 8.0 * len(sprm["blob"]) / n,
                "step_breakdown_ms": sprm["brk"], "gpu_launches": sprm["launches"],
                "cpu_baseline": cpu6}
        line = {
            "metric": METRIC, "value": value, "unit": "MB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "bytes": n,
                       "parallelism": (f"PMKLC-M over {world} GPUs: chunk c on GPU c%{world}, "
                                       "SMP handoffs as NCCL send/recv") if world > 1 else "1 GPU",
                       "l2": "256 MiB flush write between timed steps"},
            "compress_MBps": n * args.steps / 1e6 / (ct / 1000.0),
            "decompress_MBps": n * args.steps / 1e6 / (dt / 1000.0),
            "bits_per_base": 8.0 * len(blob) / n,
            "step_breakdown_ms": brk,
            "container_bytes": len(blob),
            "roofline": roof,
            "cpu_baseline": cpu,
            "sprm_branch": sprm_line,
            "e2e": {"value": e2e_val, "unit": "MB/s", "h2d_bytes_per_step": n + len(blob),
                    "d2h_bytes_per_step": len(blob) + n},
            "clocks": clk.summary(),
            "gpu_launches": launches,
        }
        print(json.dumps(line))
    if world > 1:
        torch.distributed.barrier()
        ctx.close()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
