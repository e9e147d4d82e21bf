# pass 27: round-end measurements: GPU suite, smoke, bench C2 (default) / C1 / C5, reference arm,
# C1 ncu launch list, ncu --set full of one QR-route truncation launch at C2 (dominant kernel)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu27.log 2>&1; echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke27.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > gpurun_out/bench27_c2.json 2> gpurun_out/bench27_c2.err; echo "bench c2 $?"
timeout 300 python bench.py --config 1 > gpurun_out/bench27_c1.json 2> gpurun_out/bench27_c1.err; echo "bench c1 $?"
timeout 1500 python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/bench27_c5.json 2> gpurun_out/bench27_c5.err; echo "bench c5 $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_c1.csv python bench.py --config 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu27_c1.log 2>&1; echo "ncu c1 $?"
gzip -c /tmp/launches_c1.csv > gpurun_out/r27_ncu_launches_c1.csv.gz
python tools/launch_shares.py /tmp/launches_c1.csv > gpurun_out/r27_launch_shares_c1.txt 2>&1
mkdir -p /tmp/ncu27
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_truncate<\(int\)128" -s 60 -c 2 -o /tmp/ncu27/big python tools/profile_run.py 2 > gpurun_out/ncu27_big.log 2>&1; echo "ncu big $?"
ncu -i /tmp/ncu27/big.ncu-rep --page details --csv > gpurun_out/r27_big_details.csv 2>&1
ncu -i /tmp/ncu27/big.ncu-rep --page raw --csv > gpurun_out/r27_big_raw.csv 2>&1
ncu -i /tmp/ncu27/big.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ncu27/big_src.csv 2>&1
python tools/ncu_lines.py /tmp/ncu27/big_src.csv 30 > gpurun_out/r27_big_lines.txt 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench27_ref.json 2> gpurun_out/bench27_ref.err; echo "ref $?"
