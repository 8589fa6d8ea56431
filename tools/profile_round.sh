# Round profile (run under gpurun from the repo root): bench lines, launch list, ncu --set full
# captures of the step's main kernels.  Summaries are written into profiles/ by
# tools/ncu_summary.py and tools/launch_table.py afterwards.
set -x
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
[ "$SKIP_BENCH" = 1 ] || python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
[ "$SKIP_BENCH" = 1 ] || python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
$B > gpurun_out/plain_prof.log 2>&1 || exit 1
[ "$SKIP_BENCH" = 1 ] || ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    $B > gpurun_out/ncu_l.log 2>&1
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s "$3" -c 1 \
      -o "gpurun_out/prof_$1" $B > "gpurun_out/ncu_$1.log" 2>&1
}
cap v_pre 'ozaki_pre_kernel<.bool.1>' 1
cap u_pre 'ozaki_pre_kernel<.bool.0>' 1
cap v_first 'ozaki_gemm_kernel<.bool.1' 1
cap colstats colstats 1
cap ts_gram 'gram_kernel<.int.64, .bool.1>' 4
cap ts_trmm 'mul_kernel<.int.64, .bool.1, .int.0>' 4
cap chol chol_inv_reg64 4
echo done
