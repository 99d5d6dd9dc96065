import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_1405_2270_b200.latsum import _expand_device
n = 128
out = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
fac = [torch.rand((41, n), dtype=torch.float64, device="cuda") for _ in range(3)]
w = torch.rand(41, dtype=torch.float64, device="cuda")
for _ in range(10): _expand_device(fac, w, (n, n, n), 0, n, out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200): _expand_device(fac, w, (n, n, n), 0, n, out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue per call {1e6*(t1-t0)/200:.1f} us, total per call {1e6*(t2-t0)/200:.1f} us")
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
for _ in range(200): _expand_device(fac, w, (n, n, n), 0, n, out)
e[1].record(); torch.cuda.synchronize()
print(f"GPU events per call (pipelined) {1e3*e[0].elapsed_time(e[1])/200:.1f} us")
import ctypes as C
from paper_1405_2270_b200 import _abi
lib = _abi.load()
t0 = time.perf_counter()
for _ in range(2000): lib.ls_abi_version()
t1 = time.perf_counter()
for _ in range(2000): lib.ls_expand(None, 4, None, 4, None, 4, None, 4, 4, 4, 3, 2, 5, None, 0, 0, None, None, None, None, None)
t2 = time.perf_counter()
s = torch.cuda.current_stream()
p = lambda x: C.c_void_p(x.data_ptr())
t3 = time.perf_counter()
for _ in range(200):
    lib.ls_expand(p(fac[0]), n, p(fac[1]), n, p(fac[2]), n, p(w), n, n, n, 41, 0, n, C.c_void_p(out.data_ptr()), n, n * n, None, None, None, None, C.c_void_p(s.cuda_stream))
t4 = time.perf_counter()
torch.cuda.synchronize()
t5 = time.perf_counter()
print(f"noop ctypes {1e6*(t1-t0)/2000:.2f} us, failing ls_expand {1e6*(t2-t1)/2000:.2f} us, raw ls_expand issue {1e6*(t4-t3)/200:.1f} us, total {1e6*(t5-t3)/200:.1f} us")
