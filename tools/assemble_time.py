"""CUDA-event time of estimators.assemble at c1 shape, FP64 and FP32 samples."""
import torch
from paper_2512_05749_b200 import estimators

N, P = 4096, 131072
for dt in (torch.float64, torch.float32):
    O = torch.randn(N, P, dtype=torch.float64, device="cuda").to(dt)
    E = torch.randn(N, dtype=torch.float64, device="cuda")
    batch = estimators.SampleBatch((None,) * N, E, O)
    for _ in range(2):
        estimators.assemble(batch)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        estimators.assemble(batch)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"assemble {dt}: {ms:.3f} ms  {O.numel() * O.element_size() / ms / 1e9:.2f} TB/s")
