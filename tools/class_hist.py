"""Class populations of C4 over time on the GPU (n_active histogram at checkpoints) and the
per-chunk replay time of each checkpoint interval.  usage: python tools/class_hist.py [policy]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from agft_inputs import named_config, tuner_params
from paper_2508_01744_b200 import TunerBatch
cfg = named_config("C4")
pol = int(sys.argv[1]) if len(sys.argv) > 1 else 0
tb = TunerBatch(cfg, tuner_params(cfg), device="cuda:0", policy=pol)
bins = [(1, 1), (2, 8), (9, 16), (17, 32), (33, 64), (65, 128)]
prev = 0
for T in [256, 512, 1024, 2048, 4500, 9000, 18000, 36000, 72000, 108000]:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tb.run(T, chunk=4500)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    na = tb.stats()["n_active"]
    h = [int(((na >= lo) & (na <= hi)).sum()) for lo, hi in bins]
    print(f"t={T:6d}  {dt*1e3:8.1f} ms for {T-prev:6d} steps ({dt*1e6/(T-prev):7.2f} us/step)  classes {h}", flush=True)
    prev = T
