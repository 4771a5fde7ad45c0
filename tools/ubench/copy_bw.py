import torch, time
n = 68 * 1024 * 1024 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize(); print("H2D GB/s", 10 * n * 4 / e0.elapsed_time(e1) / 1e6)
e0.record()
for _ in range(10): h2.copy_(d2, non_blocking=True)
e1.record(); torch.cuda.synchronize(); print("D2H GB/s", 10 * n * 4 / e0.elapsed_time(e1) / 1e6)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("concurrent H2D+D2H aggregate GB/s", 20 * n * 4 / dt / 1e9)
import subprocess; print(subprocess.run(["nvidia-smi", "--query-gpu=name,pcie.link.gen.current,pcie.link.width.current", "--format=csv"], capture_output=True, text=True).stdout)
