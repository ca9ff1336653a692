mkdir -p gpurun_out
rm -f /tmp/fin.ncu-rep
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:k_fin_tile -c 3 -o /tmp/fin python tools/one_exec.py ${1:-cfg5} > gpurun_out/v3_fin.log 2>&1
ncu -i /tmp/fin.ncu-rep --page raw --csv > gpurun_out/v3_fin_raw.csv 2>/dev/null
ncu -i /tmp/fin.ncu-rep --page details --csv > gpurun_out/v3_fin_details.csv 2>/dev/null
ncu -i /tmp/fin.ncu-rep --page source --csv > gpurun_out/v3_fin_source.csv 2>/dev/null
rm -f /tmp/fin.ncu-rep
