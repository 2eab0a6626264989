"""cuBLAS (torch.matmul, bf16) timings of the trainer's GEMM shapes: the library
baseline our tcgen05 kernels are compared against (warm L2, CUDA events)."""
import torch

shapes = [("fwd hidden", 1024, 2048, 2048), ("fwd out", 1024, 8806, 2048), ("dW hidden", 2048, 2048, 1024),
          ("dW out", 8806, 2048, 1024), ("dA hidden", 1024, 2048, 2048), ("dA out", 1024, 2048, 8806)]
for name, M, N, K in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        c = a @ b
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 50
    print(f"{name:12s} {M}x{N}x{K}: {us:7.2f} us  {2 * M * N * K / us / 1e6:7.1f} TFLOP/s")
