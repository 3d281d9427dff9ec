"""Drive tools/pattern_bench.cu: write GB/s of the V1 TMA tile pattern
without compute vs a coalesced STG fill, for several shapes."""
import ctypes
import json
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libpattern.so")
if not os.path.exists(so):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-shared", "-Xcompiler", "-fPIC", "-O3", "-gencode",
                           "arch=compute_100a,code=sm_100a", os.path.join(HERE, "pattern_bench.cu"), "-o", so])
L = ctypes.CDLL(so)
L.pattern_run.restype = ctypes.c_float
L.pattern_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                          ctypes.c_int, ctypes.c_int]
res = {}
for rows, n in ((2**20, 128), (2**18, 512)):
    out = torch.empty(rows * n, dtype=torch.int32, device="cuda")
    ms = L.pattern_run(1, out.data_ptr(), rows, n, 0, 0, 0, 50)
    res[f"stg_fill_{rows}x{n}"] = 4 * rows * n / ms / 1e6
    for wpb in (1, 2, 4):
        ms = L.pattern_run(3, out.data_ptr(), rows, n, 0, wpb, 0, 50)
        res[f"bulk1d_16K_{rows}x{n}_w{wpb}"] = 4 * rows * n / ms / 1e6
        ms = L.pattern_run(0, out.data_ptr(), rows, n, 32, wpb, 0, 50)
        res[f"tma2d_c32_{rows}x{n}_w{wpb}"] = 4 * rows * n / ms / 1e6
        for bands in (1, 2, 4):
            ms = L.pattern_run(2, out.data_ptr(), rows, n, bands, wpb, 0, 50)
            res[f"tma3d_b{bands}_{rows}x{n}_w{wpb}"] = 4 * rows * n / ms / 1e6
    del out
t = torch.empty(2**27, dtype=torch.int32, device="cuda")
for _ in range(3):
    t.fill_(1)
s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s_.record()
for _ in range(50):
    t.fill_(1)
e_.record()
torch.cuda.synchronize()
res["torch_fill_512MiB"] = 2**29 / (s_.elapsed_time(e_) / 50) / 1e6
print(json.dumps(res, indent=0))
