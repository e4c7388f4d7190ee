import os, sys, time, json
sys.path.insert(0, '.')
os.environ['CLTK_PLAN_CACHE'] = '0'
import paper_2108_03076_b200 as E
for kn, mn, n in [('worst-off', 'three', 16_000_000), ('european-call', 'call', 100_000_000), ('brc', 'three', 1_000_000)]:
    k = open(f'tests/golden/kernels/{kn}.json').read(); m = open(f'tests/golden/models/{mn}.json').read()
    E.price(k, m, n, 42)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); E.price(k, m, n, 42); ts.append(time.perf_counter() - t0)
    print(kn, n, 'e2e ms', [round(t * 1e3, 2) for t in ts], flush=True)
