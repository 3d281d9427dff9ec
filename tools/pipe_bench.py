"""Drive tools/pipe_bench.cu: lane-ops per clock per SM for each pipe kind
(clock = NVML SM clock sampled after the run)."""
import ctypes
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libpipe.so")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                       "arch=compute_100a,code=sm_100a", os.path.join(HERE, "pipe_bench.cu"), "-o", so])
L = ctypes.CDLL(so)
L.pipe_run.restype = ctypes.c_float
L.pipe_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
names = ["imad", "imad_hi", "lop3", "dfma", "imadhi+dfma", "imad+lop3", "ffma", "imad+ffma", "dmul",
         "dfma+lop3", "shf", "imad_wide(+lop3)"]
ops_per_chain_iter = [1, 1, 1, 1, 2, 2, 1, 2, 1, 2, 1, 2]
sms, clk = 148, 1.965e9
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    h = None
res = {}
for k, nm in enumerate(names):
    blocks, threads = sms * 8, 256
    ms = L.pipe_run(k, blocks, threads)
    if h:
        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM) * 1e6
    lane_ops = blocks * threads * 8 * L.pipe_iters() * ops_per_chain_iter[k]
    res[nm] = {"ms": ms, "lane_ops_per_clk_per_sm": lane_ops / (ms / 1e3) / clk / sms, "clk_mhz": clk / 1e6}
print(json.dumps(res, indent=1))
