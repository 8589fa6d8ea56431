# Round profile: launch list of one bench step + one ncu --set full capture of each O-pass GEMM
# kernel (v = Ohat^T q: gemm_tma_kernel<1,...>, u = Ohat v: gemm_tma_kernel<0,128,...>) + colstats.
set -x
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_prof.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Layout.1, .int.128, .int.64, .int.64" -s 4 -c 1 \
    -o gpurun_out/prof_k4 python bench.py $ARGS > gpurun_out/ncu_k4.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:Layout.0, .int.128, .int.64" -s 1 -c 1 \
    -o gpurun_out/prof_k5 python bench.py $ARGS > gpurun_out/ncu_k5.log 2>&1
echo done
