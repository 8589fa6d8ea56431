"""cuBLAS FP64 reference points (library baseline, not product): square DGEMM and the WSSR skinny shapes."""
import json, torch
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
out = {}
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
ms = t(lambda: a @ a); out["dgemm_8192_tflops"] = 2 * 8192**3 / ms / 1e9
for (N, P, k) in [(4096, 131072, 64), (16384, 131072, 128)]:
    O = torch.randn(N, P, dtype=torch.float64, device="cuda")
    q = torch.randn(P, k, dtype=torch.float64, device="cuda")
    v = torch.randn(N, k, dtype=torch.float64, device="cuda")
    ms1 = t(lambda: O @ q); ms2 = t(lambda: O.t() @ v)
    out[f"O.q_{N}x{P}x{k}_ms"] = ms1; out[f"O.q_{N}x{P}x{k}_tflops"] = 2*N*P*k/ms1/1e9
    out[f"Ot.v_{N}x{P}x{k}_ms"] = ms2; out[f"Ot.v_{N}x{P}x{k}_tflops"] = 2*N*P*k/ms2/1e9
    del O
print(json.dumps(out))
