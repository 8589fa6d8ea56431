# Profile of the c2 headline (run under gpurun from the repo root): the launch list of one bench
# step and ncu --set full captures of the step's main kernels.  Summaries are written into
# profiles/ by tools/ncu_summary.py and tools/launch_table.py afterwards.
set -x
B="python bench.py --steps 1 --warmup 3 --secondary '' --no-e2e --no-cpu-baseline"
eval "$B" > gpurun_out/plain_prof.log 2>&1 || exit 1
eval ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv "$B" > gpurun_out/ncu_l.log 2>&1
cap() {  # name regex skip
  eval ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "'regex:$2'" -s "$3" -c 1 -o "gpurun_out/prof_c2_$1" "$B" > "gpurun_out/ncu_$1.log" 2>&1
}
# on-the-fly passes at 65-128 thin columns run the transposed kernel (thin digits as A)
cap v_fly 'ozaki_gemm_t_kernel<.bool.1' 3
cap u_fly 'ozaki_gemm_t_kernel<.bool.0' 3
cap v_pre 'ozaki_pre_kernel<.bool.1' 3
cap u_pre 'ozaki_pre_kernel<.bool.0' 3
echo done
