"""Measure DFMA and DMMA (m8n8k4 f64) throughput on this GPU (roofline denominators)."""
import ctypes as C
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1602_02244_b200 import build  # noqa: E402

lib = C.CDLL(build.build_tools())
for nm in ("fp64_probe", "dmma_probe"):
    getattr(lib, nm + "_launch").argtypes = [C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    getattr(lib, nm + "_flops").argtypes = [C.c_int, C.c_int, C.c_int64]
    getattr(lib, nm + "_flops").restype = C.c_double
seed = torch.tensor([0.9999999, 1e-7, 0.5], dtype=torch.float64, device="cuda")
out = torch.zeros(1, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def rate(nm, blocks, threads, iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    rc = getattr(lib, nm + "_launch")(blocks, threads, iters, C.c_void_p(seed.data_ptr()), C.c_void_p(out.data_ptr()),
                                      C.c_void_p(st.cuda_stream))
    e1.record(st)
    e1.synchronize()
    assert rc == 0
    return getattr(lib, nm + "_flops")(blocks, threads, iters) / (e0.elapsed_time(e1) * 1e-3) / 1e12


res = {}
for nm, iters in (("fp64_probe", 20000), ("dmma_probe", 4000)):
    rate(nm, 148, 256, 100)
    for occ in (1, 2, 4, 8):
        res[f"{nm}_occ{occ}"] = max(rate(nm, 148 * occ, 256, iters) for _ in range(3))
print(json.dumps(res, indent=1))
