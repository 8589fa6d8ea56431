# Profile of the c1 secondary config (run under gpurun from the repo root): launch list of one
# bench step and ncu --set full captures of its O-pass kernels.
set -x
B="python bench.py --config c1 --steps 1 --warmup 3 --secondary '' --no-e2e --no-cpu-baseline --no-producer"
eval "$B" > gpurun_out/plain_prof_c1.log 2>&1 || exit 1
eval ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c1.csv "$B" > gpurun_out/ncu_l_c1.log 2>&1
cap() {  # name regex skip
  eval ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "'regex:$2'" -s "$3" -c 1 -o "gpurun_out/prof_c1_$1" "$B" > "gpurun_out/ncu_c1_$1.log" 2>&1
}
cap v_first 'ozaki_gemm_kernel<.bool.1' 3
cap v_pre 'ozaki_pre_kernel<.bool.1' 9
cap u_pre 'ozaki_pre_kernel<.bool.0' 12
echo done
