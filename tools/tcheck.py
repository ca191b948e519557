import sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2507_12805_b200 as P
n = 4_000_000
raw = P.synth("genome", n, 2025, 10)
cfg = P.CompressConfig(workers=128)
d = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
for i in range(4):
    t0 = time.perf_counter(); tm = P.Timing()
    b = P.compress_device(d.data_ptr(), n, cfg, tm); torch.cuda.synchronize()
    t1 = time.perf_counter()
    tm2 = P.Timing()
    ptr, ln = P.decompress_to_device(b, "", 0, tm2); torch.cuda.synchronize()
    t2 = time.perf_counter()
    P.device_free(ptr)
    t3 = time.perf_counter()
    b2 = P.compress(raw, cfg); t4 = time.perf_counter()
    x = P.decompress(b2); t5 = time.perf_counter()
    print(f"dev c {t1-t0:.3f} d {t2-t1:.3f} free {t3-t2:.3f} | host c {t4-t3:.3f} d {t5-t4:.3f} | tm.total {tm.total_ms:.1f} model {tm.model_ms:.1f} tok {tm.tokenize_ms:.1f} h2d {tm.h2d_ms:.1f}", flush=True)
