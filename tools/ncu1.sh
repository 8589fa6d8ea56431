set -x
python tools/gemm_check.py --one cm > gpurun_out/plain_cm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma -s 2 -c 1 -o gpurun_out/prof_cm python tools/gemm_check.py --one cm > gpurun_out/ncu_cm.log 2>&1
python -c "
import torch
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda')
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as p:
    b=a@a; torch.cuda.synchronize()
print(p.key_averages().table(row_limit=5))
" > gpurun_out/cublas_name.log 2>&1
