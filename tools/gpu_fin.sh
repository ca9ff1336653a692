mkdir -p gpurun_out
python tools/step_time.py cfg5 cfg3 cfg2 cfg4 2>&1 | sed 's/spec_fft.*finalize/.. finalize/'
STEP_LAYOUT=packed python tools/step_time.py cfg5 2>&1 | sed 's/spec_fft.*finalize/.. finalize/'
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/quick_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_gputest.log
tail -4 gpurun_out/quick_gputest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fin_tile -c 3 -o /tmp/fin python tools/one_exec.py cfg5 > gpurun_out/v3_fin.log 2>&1
ncu -i /tmp/fin.ncu-rep --page raw --csv > gpurun_out/v3_fin_raw.csv 2>/dev/null
ncu -i /tmp/fin.ncu-rep --page details --csv > gpurun_out/v3_fin_details.csv 2>/dev/null
ncu -i /tmp/fin.ncu-rep --page source --csv > gpurun_out/v3_fin_source.csv 2>/dev/null
