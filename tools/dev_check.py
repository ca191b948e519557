"""Developer GPU check: runs small cases through the GPU path and the oracle,
prints what matches. Not a test; used to iterate quickly under gpurun."""
import sys, time, traceback
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import paper_2507_12805_b200 as P
import oracles as O

R = O.ref() if O.REF_SO.exists() else O.port()
print("checker", R.p, "lib", P.version(), flush=True)

def step(name, fn):
    t = time.time()
    try:
        r = fn()
        print(f"[{'OK' if r else 'FAIL'}] {name} ({time.time()-t:.2f}s)", flush=True)
    except Exception as e:
        print(f"[ERR] {name}: {e}", flush=True); traceback.print_exc()

rng = np.random.default_rng(1)
def tok_check():
    ok = True
    for k in range(1, 9):
        for s in range(1, k + 1):
            n = int(rng.integers(0, 5000))
            codes = rng.integers(0, 4, n, dtype=np.uint8).tobytes()
            a = P.skmer_encode(codes, s, k); b, _ = R.skmer_encode(codes, s, k)
            if not np.array_equal(a, b): ok = False; print("tok mismatch", s, k, n)
    return ok
step("tokenizer 36 (s,k)", tok_check)

def dump_check():
    raw = P.synth("markov3", 30000, 3)
    codes = bytes(((b >> 1) ^ (b >> 2)) & 3 for b in raw)
    tok, _ = R.skmer_encode(codes, 3, 3)
    n = 16 * 40
    pa, sa, pr_ref = R.dump_chunk(tok[:n], 4, 3, 8, 16, 16, 1234, max_steps=32)
    pb, pr_gpu = P.dump_chunk(tok[:n], 4, 3, 8, 16, 16, 1234, max_steps=32)
    eq = np.array_equal(pr_ref.view(np.uint32), pr_gpu.view(np.uint32))
    if not eq:
        d = np.abs(pr_ref - pr_gpu)
        for s in range(pr_ref.shape[0]):
            if d[s].max() > 0: print("first diff step", s, d[s].max()); break
    print("payload eq", pa == pb, len(pa), len(pb))
    return eq and pa == pb
step("dump chunk probs bitwise (t=8,bs=16,scale16)", dump_check)

def cont(raw, **kw):
    c = P.CompressConfig(**{k: v for k, v in kw.items() if k != 'smp'}, **({'smp_fraction': kw['smp']} if 'smp' in kw else {}))
    t = time.time(); a = P.compress(raw, c); tg = time.time() - t
    b = R.compress(raw, O.make_cfg(**kw))
    rt = P.decompress(a) == raw
    print(f"   len gpu={len(a)} ref={len(b)} eq={a==b} rt={rt} gpu {tg:.2f}s", flush=True)
    return a == b and rt
step("uniform fixture t=4096", lambda: cont(P.synth("uniform", 12000, 9), t=4096))
step("small W=1", lambda: cont(P.synth("markov3", 20000, 1), t=4, bs=16, scale=16))
step("small W=3 smp", lambda: cont(P.synth("markov3", 50000, 2), t=8, bs=64, scale=16, workers=3))
step("k=1 W=2", lambda: cont(P.synth("markov3", 20000, 5), s=1, k=1, t=4, bs=16, scale=16, workers=2, smp=0.1))
step("k=4 s=2", lambda: cont(P.synth("markov3", 20000, 6), s=2, k=4, t=4, bs=16, scale=16, workers=2, smp=0.1))
step("exceptions", lambda: cont(P.synth("markov3", 20000, 8) + b"NNacgt>\nACGT", t=4, bs=16, scale=16))
if len(sys.argv) > 1 and sys.argv[1] == "big":
    raw = P.synth("markov3", 1 << 20, 12345)
    c = P.CompressConfig(workers=8)
    st = P.PipelineStats()
    t = time.time(); a = P.compress(raw, c, st); tg = time.time() - t
    print("W=8 len", len(a), hex(O.fnv1a64(a)), "want 254517 0x60402d686aefd79d", f"{tg:.2f}s", st.timing.model_ms, st.timing.ticks)
    c = P.CompressConfig()
    t = time.time(); a = P.compress(raw, c, st); tg = time.time() - t
    print("W=1 len", len(a), hex(O.fnv1a64(a)), "want 231207 0xc59806701e845e33", f"{tg:.2f}s", st.timing.model_ms, st.timing.ticks)
    t = time.time(); d = P.decompress(a, stats=st); td = time.time() - t
    print("W=1 decompress ok", d == raw, f"{td:.2f}s", st.timing.model_ms)
