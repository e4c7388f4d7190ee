import sys, json, time
sys.setrecursionlimit(100000); sys.path.insert(0, '.')
import paper_2108_03076_b200 as E
k = json.load(open('tests/golden/kernels/worst-off.json')); m = json.load(open('tests/golden/models/three.json'))
import torch; torch.cuda.init()
for jit in (False, True):
    for rep in range(4):
        t = time.perf_counter(); E.price(k, m, 16_000_000, 42, jit=jit); t1 = time.perf_counter() - t
        t = time.perf_counter(); p = E.Plan(E.Kernel(k), m, [0], jit=jit); t2 = time.perf_counter() - t
        t = time.perf_counter(); E.price(k, m, 1000, 42, jit=jit); t3 = time.perf_counter() - t
        print(f"jit={jit} rep={rep} price16M {t1*1e3:.1f} ms  plan {t2*1e3:.1f} ms  price1k {t3*1e3:.1f} ms", flush=True)
