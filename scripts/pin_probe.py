import sys, time, ctypes as C
sys.path.insert(0, ".")
import paper_1805_08995_b200 as ch
from paper_1805_08995_b200 import _native as N
with ch.Matcher(0) as m:
    lib = N.load()
    for mb in (16, 160, 320, 640):
        p = C.c_void_p()
        t0 = time.perf_counter(); st = lib.chgpu_host_alloc(m.h, mb << 20, C.byref(p)); t1 = time.perf_counter()
        lib.chgpu_host_free(m.h, p); t2 = time.perf_counter()
        print(f"cudaMallocHost {mb} MiB: {1e3*(t1-t0):.1f} ms, free {1e3*(t2-t1):.1f} ms, status {st}")
