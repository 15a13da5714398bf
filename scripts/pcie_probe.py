import torch, time
n = 52 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s = torch.cuda.Stream()
for _ in range(3):
    with torch.cuda.stream(s): h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10):
    with torch.cuda.stream(s): h.copy_(d, non_blocking=True)
e1.record(s); torch.cuda.synchronize()
print("contiguous D2H GB/s", 10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
# 2-D: 700 rows of 600*128 B out of a 1024*128 B pitch
import ctypes
cudart = ctypes.CDLL("libcudart.so")
W = 1024 * 128; w = 600 * 128; rows = 700
dd = torch.empty(W * rows, dtype=torch.uint8, device="cuda"); hh = torch.empty(W * rows, dtype=torch.uint8, pin_memory=True)
fn = cudart.cudaMemcpy2DAsync
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
e0.record(s)
for _ in range(10):
    fn(hh.data_ptr(), W, dd.data_ptr(), W, w, rows, 2, ctypes.c_void_p(s.cuda_stream))
e1.record(s); torch.cuda.synchronize()
print("2D D2H GB/s", 10 * w * rows / (e0.elapsed_time(e1) / 1e3) / 1e9)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
e0.record(s)
for _ in range(10):
    with torch.cuda.stream(s): d.copy_(h2, non_blocking=True)
e1.record(s); torch.cuda.synchronize()
print("contiguous H2D GB/s", 10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
# the frame stream's box readout: F rows of 128 B/pixel, A/D rows of 4 B/pixel
for per in (128, 4):
    Wp = 1024 * per; wb = 640 * per; rows = 720
    dd = torch.empty(Wp * 1024, dtype=torch.uint8, device="cuda"); hh = torch.empty(Wp * 1024, dtype=torch.uint8, pin_memory=True)
    e0.record(s)
    for _ in range(10):
        fn(hh.data_ptr(), Wp, dd.data_ptr(), Wp, wb, rows, 2, ctypes.c_void_p(s.cuda_stream))
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"2D D2H {per} B/px: {ms:.3f} ms per copy, {wb * rows / ms / 1e6:.1f} GB/s")
