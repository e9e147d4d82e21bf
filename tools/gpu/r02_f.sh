# DMMA solve kernels: solve roofline at C2 / C5, then the full GPU suite
mkdir -p gpurun_out
timeout 300 python tools/solve_bench.py 2 - 5 > gpurun_out/solve_c2_f.json 2>&1
timeout 900 python tools/solve_bench.py 5 - 3 > gpurun_out/solve_c5_f.json 2>&1
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_f.log
