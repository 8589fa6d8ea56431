# ncu of the CholeskyQR2 tall-skinny GEMMs at c1 shape (Gram: CM 64x64xP, TRMM: RM Px64x64)
PYTHONPATH=. python tools/ts_time.py > gpurun_out/ts_plain.log 2>&1 || exit 1
PYTHONPATH=. ncu --set full --clock-control none -k regex:gemm_tma_kernel -s 4 -c 2 -o gpurun_out/prof_ts python tools/ts_time.py > gpurun_out/ncu_ts.log 2>&1
cat gpurun_out/ts_plain.log
