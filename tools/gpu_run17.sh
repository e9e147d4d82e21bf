# pass 17: ncu --set full of the reworked small kernels (text summaries only come back) + PCG time-to-solution
set -x
mkdir -p /tmp/ncu17
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_small32<\(int\)1>" -s 300 -c 1 -o /tmp/ncu17/dd32 python tools/profile_run.py 2 > gpurun_out/ncu17a.log 2>&1; echo "a $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_truncate<\(int\)64" -s 100 -c 1 -o /tmp/ncu17/mid64 python tools/profile_run.py 2 > gpurun_out/ncu17b.log 2>&1; echo "b $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_truncate<\(int\)128" -s 60 -c 2 -o /tmp/ncu17/big python tools/profile_run.py 2 > gpurun_out/ncu17c.log 2>&1; echo "c $?"
for r in dd32 mid64 big; do
  ncu -i /tmp/ncu17/$r.ncu-rep --page details --csv > gpurun_out/r17_${r}_details.csv 2>&1
  ncu -i /tmp/ncu17/$r.ncu-rep --page raw --csv > gpurun_out/r17_${r}_raw.csv 2>&1
  ncu -i /tmp/ncu17/$r.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ncu17/${r}_src.csv 2>&1
  python tools/ncu_lines.py /tmp/ncu17/${r}_src.csv 30 > gpurun_out/r17_${r}_lines.txt 2>&1
done
ls -la gpurun_out/
timeout 600 python tools/pcg_run.py 2 1e-2 1e-8 > gpurun_out/pcg_c2.json 2> gpurun_out/pcg_c2.err; echo "pcg c2 $?"
