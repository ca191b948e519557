"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections, csv, re, sys

def main(fn, ticks=None):
    rows = list(csv.reader(open(fn)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]; data = rows[hi + 1:]
    ki, vi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
    agg = collections.defaultdict(list)
    for r in data:
        name = r[ki]
        m = re.search(r'(k_\w+)', name); n = m.group(1) if m else name[:40]
        if 'k_gemm_tiled' in n:
            n = 'gemm<' + re.search(r'k_gemm_tiled<([^>]*)>', name).group(1) + '> ' + r[gi]
        agg[n].append(float(r[vi].replace(',', '')) / 1000)
    tot = sum(sum(v) for v in agg.values())
    for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{sum(v):9.1f} us {100*sum(v)/tot:5.1f}%  n={len(v):3d} avg={sum(v)/len(v):8.1f}  {n}")
    print(f"total {tot:.1f} us over {len(data)} launches")

if __name__ == '__main__':
    main(sys.argv[1])
