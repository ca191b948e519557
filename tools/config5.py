"""BASELINE config 5 at N=1, scaled (one-off measurement, not the bench default).

Config 5 is a 10 GB multi-species mixture with distribution-perturbed blocks on
8 GPUs. One GPU gets 1/8 of it under PMKLC-M, so this runs a 1/10 sample
(10^9 B by default) of the same structure: `synth_species` with the switching
block shrunk by the same factor, so the sample still holds 160 source blocks,
every 16th drawn from a perturbed table (csrc/host/synth.cpp). Default selector
(> 500 MB => SPrM pre-pass + DM, flags 6), W=256, defaults otherwise.

Robustness: per-chunk bits/base from the container's chunk table, split into
chunks lying inside perturbed source blocks and the rest. Device-resident
input; compress and decompress timed with CUDA events; lossless round trip
checked through the host API."""
import json
import struct
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2507_12805_b200 as P

n = int(float(sys.argv[1]) * 1e6) if len(sys.argv) > 1 else 10**9
W = int(sys.argv[2]) if len(sys.argv) > 2 else 256
# source block: 160 of them as in the 10 GB config (default), or a given size
# (64 MiB = the 10 GB config's own blocks, for a contiguous 1/8 share)
block = int(sys.argv[3]) if len(sys.argv) > 3 else max(1, int((64 << 20) * n / 1e10))
t0 = time.time()
raw = P.synth("species", n, 2026, block)
cfg = P.CompressConfig(workers=W, max_workers=max(W, 256))
d_raw = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
tc, td = P.Timing(), P.Timing()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
torch.cuda.synchronize()
e[0].record()
blob = P.compress_device(d_raw.data_ptr(), n, cfg, tc)
e[1].record()
torch.cuda.synchronize()
e[2].record()
dptr, dlen = P.decompress_to_device(blob, "", 0, td)
e[3].record()
torch.cuda.synchronize()
out = P.decompress(blob, "")  # host API round trip check
ok = out == raw
P.device_free(dptr)
c_ms, d_ms = e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])

# chunk table: 52-byte header (W at 48), 36-byte entries (token_start, token_len,
# offset, payload_len u64; trailer_len u32) -- container.cpp write_container
s = blob[6]
nchunks = struct.unpack_from("<I", blob, 48)[0]
pert_bits = pert_bases = norm_bits = norm_bases = 0
per_chunk = []
for i in range(nchunks):
    ts, tl, _, pl, tr = struct.unpack_from("<QQQQI", blob, 52 + 36 * i)
    b0, nb = ts * s, tl * s
    if nb == 0:
        continue
    first, last = b0 // block, (b0 + nb - 1) // block
    bpb = 8 * (pl + tr) / nb
    kind = "mixed"
    if first == last:
        kind = "perturbed" if first % 16 == 15 else "normal"
    per_chunk.append(round(bpb, 4))
    if kind == "perturbed":
        pert_bits += 8 * (pl + tr)
        pert_bases += nb
    elif kind == "normal":
        norm_bits += 8 * (pl + tr)
        norm_bases += nb
print(json.dumps({
    "config": "config5 sample (N=1): species mixture, %d source blocks of %d B, every 16th perturbed"
              % ((n + block - 1) // block, block),
    "bytes": n, "W": W, "container_flags": blob[5],
    "compress_MBps": n / 1e6 / (c_ms / 1e3), "decompress_MBps": n / 1e6 / (d_ms / 1e3),
    "round_trip_MBps": n / 1e6 / ((c_ms + d_ms) / 1e3), "bits_per_base": 8 * len(blob) / n,
    "bits_per_base_normal_chunks": norm_bits / max(norm_bases, 1),
    "bits_per_base_perturbed_chunks": pert_bits / max(pert_bases, 1),
    "chunks_normal_bases": norm_bases, "chunks_perturbed_bases": pert_bases,
    "crp_percent_blocks": P.robustness(P.block_ratios(blob)),
    "state_tape_slots": tc.slots, "device_peak_bytes_compress": tc.dev_peak_bytes,
    "device_peak_bytes_decompress": td.dev_peak_bytes,
    "sprm_prepass_ms": tc.sprm_ms, "compress_ticks_ms": tc.model_ms,
    "decompress_ticks_ms": td.model_ms, "ticks": tc.ticks, "lossless": ok,
    "wall_s": time.time() - t0, "per_chunk_bits_per_base": per_chunk}))
