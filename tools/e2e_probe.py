"""Where the end-to-end time of one public-API call goes (run under gpurun):
   python tools/e2e_probe.py [kernel] [model] [paths]"""
import sys, json, time
sys.setrecursionlimit(100000); sys.path.insert(0, '.')
import paper_2108_03076_b200 as E
kn = sys.argv[1] if len(sys.argv) > 1 else 'brc'
mn = sys.argv[2] if len(sys.argv) > 2 else 'three'
paths = int(float(sys.argv[3])) if len(sys.argv) > 3 else 125_000_000
k = open(f'tests/golden/kernels/{kn}.json').read(); m = open(f'tests/golden/models/{mn}.json').read()
import torch; torch.cuda.init()
E.price(k, m, 1000, 42, jit=True)  # NVRTC module cache
for rep in range(3):
    t = time.perf_counter(); E.price(k, m, paths, 42, jit=True); t1 = time.perf_counter() - t
    t = time.perf_counter(); p = E.Plan(E.Kernel(k), m, [0], jit=True); t2 = time.perf_counter() - t
    t = time.perf_counter(); E.price(k, m, 1000, 42, jit=True); t3 = time.perf_counter() - t
    t = time.perf_counter(); kk = E.Kernel(k); t4 = time.perf_counter() - t
    nc = p.chunking(paths)
    t = time.perf_counter(); parts = torch.zeros(nc[1] * p.n_outputs * 3, dtype=torch.float64, device='cuda')
    s = torch.cuda.current_stream()
    p.launch(paths, 42, 0, nc[1], parts.data_ptr(), s.cuda_stream); torch.cuda.synchronize(); t5 = time.perf_counter() - t
    print(f"rep={rep} price({paths:.3g}) {t1*1e3:.1f} ms | Plan() {t2*1e3:.1f} ms | price(1k) {t3*1e3:.1f} ms | "
          f"Kernel() {t4*1e3:.1f} ms | launch only {t5*1e3:.1f} ms", flush=True)
