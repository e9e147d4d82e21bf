# pass 32: tile-GEMM staging loads grouped ahead of smem stores; GPU suite, C2 levels, final bench lines C2/C1
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu32.log 2>&1; echo "pytest exit $?"
ACRGPU_VERBOSE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof32_c2_levels_np.log 2>&1
ACRGPU_VERBOSE=1 ACRGPU_PROFILE=1 timeout 300 python tools/profile_run.py 2 > gpurun_out/prof32_c2_levels.log 2>&1
timeout 600 python bench.py > gpurun_out/bench32_c2.json 2> gpurun_out/bench32_c2.err; echo "bench c2 $?"
timeout 300 python bench.py --config 1 > gpurun_out/bench32_c1.json 2> gpurun_out/bench32_c1.err; echo "bench c1 $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke32.log 2>&1; echo "smoke exit $?"
