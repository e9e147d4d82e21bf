# pass 19 (session re-entry): GPU suite, smoke, bench lines at the current commit, reference arm
set -x
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu19.log 2>&1; echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke19.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > gpurun_out/bench19_c2.json 2> gpurun_out/bench19_c2.err; echo "bench c2 $?"
timeout 300 python bench.py --config 1 > gpurun_out/bench19_c1.json 2> gpurun_out/bench19_c1.err; echo "bench c1 $?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench19_ref.json 2> gpurun_out/bench19_ref.err; echo "ref $?"
