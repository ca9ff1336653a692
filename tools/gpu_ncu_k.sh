# bash tools/gpu_ncu_k.sh <kernel regex> <cfg> <tag> [count]
mkdir -p gpurun_out
rm -f /tmp/k.ncu-rep
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$1 -c ${4:-1} -o /tmp/k python tools/one_exec.py $2 > gpurun_out/$3.log 2>&1
ncu -i /tmp/k.ncu-rep --page raw --csv > gpurun_out/$3_raw.csv 2>/dev/null
ncu -i /tmp/k.ncu-rep --page details --csv > gpurun_out/$3_details.csv 2>/dev/null
ncu -i /tmp/k.ncu-rep --page source --csv > gpurun_out/$3_source.csv 2>/dev/null
rm -f /tmp/k.ncu-rep
