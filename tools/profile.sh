# Round profile: one ncu --set full capture of each O-pass kernel (v = Ohat^T q:
# ozaki_pre_kernel<1>, u = Ohat v: ozaki_pre_kernel<0>), the per-step digitising pass and the
# assemble column pass.  Run under gpurun from the repo root.
set -x
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_prof.log 2>&1 || exit 1
# ozaki_pre_kernel launches alternate v = Ohat^T q (row-major pass) and u = Ohat v
ncu --set full --clock-control none --import-source on -k regex:ozaki_pre_kernel -s 8 -c 1 \
    -o gpurun_out/prof_k4 python bench.py $ARGS > gpurun_out/ncu_k4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ozaki_pre_kernel -s 9 -c 1 \
    -o gpurun_out/prof_k5 python bench.py $ARGS > gpurun_out/ncu_k5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:digitize -s 3 -c 1 \
    -o gpurun_out/prof_dg python bench.py $ARGS > gpurun_out/ncu_dg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:colstats -s 3 -c 1 \
    -o gpurun_out/prof_cs python bench.py $ARGS > gpurun_out/ncu_cs.log 2>&1
echo done
