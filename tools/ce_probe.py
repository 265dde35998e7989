"""Copy-engine contention probe: does a small copy on one stream wait behind a
bulk pinned H2D copy on another stream (whole, or issued in 8 MB chunks)?"""
import time

import numpy as np
import torch

dev = torch.device("cuda:0")
big_h = torch.empty(466 * 2**20 // 8, dtype=torch.float64).pin_memory()
big_d = torch.empty_like(big_h, device=dev)
small_np = np.ones(4 * 2**20, np.uint8)
small_pin = torch.from_numpy(small_np).pin_memory()
small_d = torch.empty(4 * 2**20, dtype=torch.uint8, device=dev)
tiny_d = torch.ones(1024, dtype=torch.float64, device=dev)
tiny_h = torch.empty(1024, dtype=torch.float64).pin_memory()
s_bulk = torch.cuda.Stream()
s_work = torch.cuda.Stream()


def bulk(chunked):
    with torch.cuda.stream(s_bulk):
        if not chunked:
            big_d.copy_(big_h, non_blocking=True)
        else:
            step = 8 * 2**20 // 8
            for i in range(0, big_h.numel(), step):
                big_d[i:i + step].copy_(big_h[i:i + step], non_blocking=True)


for chunked in (False, True):
    for trial in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bulk(chunked)
        t1 = time.perf_counter()
        with torch.cuda.stream(s_work):
            tiny_h.copy_(tiny_d, non_blocking=True)
            s_work.synchronize()
        t2 = time.perf_counter()
        with torch.cuda.stream(s_work):
            small_d.copy_(small_pin, non_blocking=True)
            s_work.synchronize()
        t3 = time.perf_counter()
        s_bulk.synchronize()
        t4 = time.perf_counter()
        print(f"chunked={chunked}: issue {1e3*(t1-t0):.2f} ms, tiny D2H {1e3*(t2-t1):.2f} ms, "
              f"pinned 4MB H2D {1e3*(t3-t2):.2f} ms, bulk done {1e3*(t4-t0):.2f} ms")
