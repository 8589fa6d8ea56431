set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_implicit_dense.py tests/test_gpu_sharded_emulated.py -x -q -s --durations=10 > gpurun_out/t2.log 2>&1
echo tests rc $?
B="python bench.py --steps 5 --warmup 3 --secondary '' --no-e2e --no-cpu-baseline"
WSSR_OZ_TKERNEL=1 timeout 600 bash -c "$B" > gpurun_out/b_t1.json 2> gpurun_out/b_t1.err
echo b1 rc $?
WSSR_OZ_TKERNEL=2 timeout 600 bash -c "$B" > gpurun_out/b_t2.json 2> gpurun_out/b_t2.err
echo b2 rc $?
