"""Host<->device transfer paths on the bench box (bounds the e2e host-buffer
SpMV: 4 MB of x in and 4 MB of y out per C2 step).  Pinned host buffers.

  ce_h2d / ce_d2h   copy engine (cudaMemcpyAsync) per size
  sm_read / sm_write  knnx_copy_async: SMs load from / store to mapped host
                      memory (zero-copy, no copy engine)
  ce_h2d+sm_write   both directions at once (the pipelined e2e pattern)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1709_03671_b200 import api
from paper_1709_03671_b200._lib import check, lib

ctx = api.Context(0)
s_main = torch.cuda.Stream()
ctx.use_stream(s_main)
s_ce = torch.cuda.Stream()
out = {}


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_main)
    s_ce.wait_event(e0)
    for _ in range(reps):
        fn()
    s_main.wait_stream(s_ce)
    e1.record(s_main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


for mb in (1, 4, 16, 64):
    nb = mb << 20
    hx = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
    hy = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
    dx = torch.empty(nb // 4, device="cuda")
    dy = torch.empty(nb // 4, device="cuda")
    reps = max(5, 200 // mb)

    def ce_h2d():
        with torch.cuda.stream(s_ce):
            dx.copy_(hx, non_blocking=True)

    def ce_d2h():
        with torch.cuda.stream(s_ce):
            hy.copy_(dy, non_blocking=True)

    def sm_read():
        check(lib.knnx_copy_async(ctx.h, C.c_void_p(dx.data_ptr()), C.c_void_p(hx.data_ptr()), nb))

    def sm_write():
        check(lib.knnx_copy_async(ctx.h, C.c_void_p(hy.data_ptr()), C.c_void_p(dy.data_ptr()), nb))

    def both():
        ce_h2d()
        sm_write()

    rec = {}
    for name, fn in (("ce_h2d", ce_h2d), ("ce_d2h", ce_d2h), ("sm_read", sm_read),
                     ("sm_write", sm_write), ("ce_h2d+sm_write", both)):
        us = timed(fn, reps)
        rec[name + "_us"] = round(us, 1)
        rec[name + "_GBs"] = round(nb * (2 if name == "ce_h2d+sm_write" else 1) / us / 1e3, 1)
    out[f"{mb}MB"] = rec
    print(mb, rec, flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/pcie.json", "w") as f:
    json.dump(out, f, indent=1)
