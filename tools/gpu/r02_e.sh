# memcheck of the new paths (fork/join mult_add, async gc, two-phase solve), full GPU suite, A/B timing
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/factor_time.py 2 8 1 > gpurun_out/memcheck_c2n8.log 2>&1; echo rc=$? >> gpurun_out/memcheck_c2n8.log
ACRGPU_GC_FORCE=0.000001 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/factor_time.py 5 4 1 > gpurun_out/memcheck_c5n4.log 2>&1; echo rc=$? >> gpurun_out/memcheck_c5n4.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_e.log 2>&1; echo rc=$? >> gpurun_out/pytest_e.log
timeout 300 python tools/factor_time.py 2 - 3 > gpurun_out/ft_c2_e.jsonl 2>&1
timeout 600 python tools/factor_time.py 5 - 1 > gpurun_out/ft_c5_e.jsonl 2>&1
