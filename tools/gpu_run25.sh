# pass 25: ncu --set full of one top-level (level 6) k_small32<1> launch and one level-1 launch, source hot spots
set -x
mkdir -p /tmp/ncu25
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_small32<\(int\)1>" -s 4900 -c 1 -o /tmp/ncu25/top python tools/profile_run.py 2 > gpurun_out/ncu25a.log 2>&1; echo "a $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_small32<\(int\)1>" -s 1000 -c 1 -o /tmp/ncu25/l1 python tools/profile_run.py 2 > gpurun_out/ncu25b.log 2>&1; echo "b $?"
for r in top l1; do
  ncu -i /tmp/ncu25/$r.ncu-rep --page details --csv > gpurun_out/r25_${r}_details.csv 2>&1
  ncu -i /tmp/ncu25/$r.ncu-rep --page raw --csv > gpurun_out/r25_${r}_raw.csv 2>&1
  ncu -i /tmp/ncu25/$r.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ncu25/${r}_src.csv 2>&1
  python tools/ncu_lines.py /tmp/ncu25/${r}_src.csv 40 > gpurun_out/r25_${r}_lines.txt 2>&1
  cp /tmp/ncu25/$r.ncu-rep gpurun_out/ 2>/dev/null
done
