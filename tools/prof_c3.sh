# ncu --set full capture of one pre-digitised O-pass at c3 (5-digit planes), after 3 warm-up steps
B=(python bench.py --config c3 --secondary "" --no-e2e --no-cpu-baseline --steps 1 --warmup 3)
"${B[@]}" > gpurun_out/plain_c3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:ozaki_pre_kernel -s 21 -c 2 \
    -o gpurun_out/prof_c3_pre "${B[@]}" > gpurun_out/ncu_c3.log 2>&1
