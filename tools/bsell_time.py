import sys, time, ctypes
sys.path.insert(0, '.')
import numpy as np
from paper_1801_08464_b200 import _lib, synth
from paper_1801_08464_b200.sparse import DeviceMatrix, block_scale
s = synth.make_config(3, 128)
ctx = _lib.ctx()
n = s.n
x = _lib.P(); y = _lib.P()
ctx.call("mg_dev_alloc", 8 * n, ctypes.byref(x)); ctx.call("mg_dev_alloc", 8 * n, ctypes.byref(y))
for rep in range(3):
    d = DeviceMatrix.from_bsr(s.rowptr, s.col, s.vals, ctx=ctx)
    ctx.sync()
    t0 = time.perf_counter(); ctx.call("mg_spmv_dev", d.h, x, y); ctx.sync(); t1 = time.perf_counter()
    ctx.call("mg_spmv_dev", d.h, x, y); ctx.sync(); t2 = time.perf_counter()
    t3 = time.perf_counter(); dv, ah = block_scale(d); ctx.sync(); t4 = time.perf_counter()
    print(f"first spmv (BSELL build + spmv) {1e3*(t1-t0):.2f} ms, second {1e3*(t2-t1):.3f} ms, block_scale {1e3*(t4-t3):.2f} ms")
    dv.free(); ah.free(); d.free()
