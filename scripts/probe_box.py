"""Host/PCIe/tensor-core probes for the roofline denominators (run on the GPU box)."""
import json, os, time
import torch
out = {}
out["cpu_count"] = os.cpu_count()
try:
    with open("/proc/meminfo") as f:
        out["mem_total_gb"] = int(f.readline().split()[1]) / 1e6
except Exception:
    pass
dev = torch.device("cuda:0")
# pinned H2D / D2H bandwidth (1 GiB)
n = 1 << 28
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device=dev)
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    out[f"pinned_{name}_gbs"] = n * 4 / best / 1e9
# cuBLAS TF32 and FP32 GEMM throughput (8192^3)
a = torch.randn(8192, 8192, device=dev)
b = torch.randn(8192, 8192, device=dev)
for name, tf32 in (("tf32", True), ("fp32_simt", False)):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.matmul(a, b); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); torch.matmul(a, b); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    out[f"cublas_{name}_tflops"] = 2 * 8192 ** 3 / best / 1e12
ad = a.double(); bd = b.double()
torch.matmul(ad, bd); torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); torch.matmul(ad, bd); e.record(); torch.cuda.synchronize()
out["cublas_fp64_tflops"] = 2 * 8192 ** 3 / (s.elapsed_time(e) / 1e3) / 1e12
print(json.dumps(out))
