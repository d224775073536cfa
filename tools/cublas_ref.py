"""cuBLAS (torch.matmul) times for the C2 GEMM shapes, for comparison with
the hand-written kernels (not used by the product)."""
import torch

shapes = {"qkv": (4096, 3456, 1152), "out_proj": (4096, 1152, 1152),
          "mlp_in": (4096, 4608, 1152), "mlp_out": (4096, 1152, 4608),
          "out_proj_r512": (512, 1152, 1152), "mlp_out_r512": (512, 1152, 4608)}
for name, (m, n, k) in shapes.items():
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(m, n, device="cuda", dtype=torch.float32)
    for _ in range(10):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    print(f"{name:14s} {m}x{n}x{k}: {us:7.2f} us  {2 * m * n * k / us / 1e6:7.1f} TF/s")
