import os, sys, time
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.getcwd())
import torch
import paper_1610_05108_b200 as xb
from paper_1610_05108_b200 import synth, _lib
x, y, _ = synth.gwas()
pin = torch.empty(x.words.nbytes, dtype=torch.uint8, pin_memory=True)
pw = pin.numpy().view(x.words.dtype).reshape(x.words.shape); pw[...] = x.words
xh = xb.PackedMatrix(x.n_rows, x.n_cols, pw)
cfg = xb.SearchConfig(m=16, l=100, gamma=0.6, seed=7, top_k=100, estimate_complexity=False, top_k_mode="candidates")
def step(i):
    d = xb.Dataset(xh); r = d.search(y, cfg); d.close(); return r
with ThreadPoolExecutor(4) as ex:
    list(ex.map(step, range(16)))
    torch.cuda.synchronize()
    _lib.set_test_option("trace", 1)
    print("=== traced", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    list(ex.map(step, range(16)))
    torch.cuda.synchronize()
    _lib.set_test_option("trace", 0)
    print(f"{1e3*(time.perf_counter()-t0)/16:.3f} ms/step", file=sys.stderr, flush=True)
