"""HBM streaming calibration: torch reductions / cuBLAS GEMV at the decode
weight sizes, to separate per-kernel fixed cost from streaming rate (run under
ncu --metrics gpu__time_duration.sum)."""
import torch
dev = torch.device("cuda", 0)
for K, N in ((4096, 4096), (4096, 6144), (4096, 14336), (4096, 28672)):
    W = torch.randn(K, N, device=dev).to(torch.bfloat16)
    A = torch.randn(1, K, device=dev).to(torch.bfloat16)
    for _ in range(3):
        W.sum(dtype=torch.float32)
        torch.matmul(A, W)
    torch.cuda.synchronize()
    del W, A
