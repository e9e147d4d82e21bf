# pass 10: C5 bench line (one factorization + 16-RHS solve per step)
set -x
timeout 1500 python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 exit $?"
