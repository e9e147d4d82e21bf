# pass 34: final bench lines (C2 default, C1, C5) at the deposit change, C1 ncu launch list, smoke
set -x
timeout 600 python bench.py > gpurun_out/bench34_c2.json 2> gpurun_out/bench34_c2.err; echo "bench c2 $?"
timeout 300 python bench.py --config 1 > gpurun_out/bench34_c1.json 2> gpurun_out/bench34_c1.err; echo "bench c1 $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke34.log 2>&1; echo "smoke exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_c1.csv python bench.py --config 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu34_c1.log 2>&1; echo "ncu c1 $?"
gzip -c /tmp/launches_c1.csv > gpurun_out/r34_ncu_launches_c1.csv.gz
python tools/launch_shares.py /tmp/launches_c1.csv > gpurun_out/r34_launch_shares_c1.txt 2>&1
timeout 1500 python bench.py --config 5 --steps 1 --warmup 3 > gpurun_out/bench34_c5.json 2> gpurun_out/bench34_c5.err; echo "bench c5 $?"
