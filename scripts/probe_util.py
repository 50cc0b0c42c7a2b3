"""NVML GPU utilisation (fraction of sample periods with a kernel running) and
SM clock during repeated sweep shares -- is the sweep GPU-bound or host-bound?"""
import sys, threading, time
sys.path.insert(0, ".")
import pynvml
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
s = [x for x in sweep_samples() if x["id"] % 8 == 0]
hh.sweep(s)
util, stop = [], [False]
def sampler():
    while not stop[0]:
        u = pynvml.nvmlDeviceGetUtilizationRates(h)
        util.append(u.gpu)
        time.sleep(0.02)
th = threading.Thread(target=sampler); th.start()
t0 = time.perf_counter()
for _ in range(10):
    hh.sweep(s)
dt = time.perf_counter() - t0
stop[0] = True; th.join()
print(f"10 sweeps {dt:.2f} s, NVML util mean {sum(util)/len(util):.1f}% over {len(util)} samples, min {min(util)}")
