"""Summarise an ncu launch list (gpu__time_duration) of bench.py: per-kernel
time of the last timed step (the last 32 attention launches of the main
measurement and the pool/engine kernels around them)."""
import collections
import csv
import sys


def main(path, n_layers=32, steps_before=3):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    data = rows[hi + 1:]
    att = [i for i, r in enumerate(data) if 'k_continuation_attention' in r[ki]]
    k = steps_before  # step index (0-based) of the timed step
    s0 = att[k * n_layers - 1] + 1 if k else 0
    e = att[(k + 1) * n_layers - 1] + 1
    while e < len(data) and data[e][ki].startswith(('sb::', 'void sb', '<unnamed>', 'attn')) and \
            'k_chain_hash16' not in data[e][ki]:
        e += 1
    seg = data[s0:e]
    agg = collections.OrderedDict()
    tot = 0.0
    for r in seg:
        name = r[ki].split('(')[0][:48]
        v = float(r[vi].replace(',', ''))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    for name, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name:48s} {n:4d} {v / 1e3:10.1f} us  {100 * v / tot:5.2f} %")
    print(f"step {tot / 1e6:.2f} ms (serialised, cold); sequence:")
    print([(r[ki].split('(')[0].replace('void ', '')[:22], round(float(r[vi].replace(',', '')) / 1e3, 1))
           for r in seg if 'attention' not in r[ki] and 'append' not in r[ki]])


if __name__ == "__main__":
    main(sys.argv[1])
