mkdir -p gpurun_out
echo "== default (minB 2, single stage)"; python tools/step_time.py cfg5 cfg4 2>&1 | sed 's/spec_fft.*finalize/.. finalize/'
echo "== a (minB 1, double stage)"; COVGPU_LIB=$PWD/gpurun_var_a.so python tools/step_time.py cfg5 2>&1 | sed 's/spec_fft.*finalize/.. finalize/'
echo "== b (minB 1, single stage)"; COVGPU_LIB=$PWD/gpurun_var_b.so python tools/step_time.py cfg5 2>&1 | sed 's/spec_fft.*finalize/.. finalize/'
STEP_LAYOUT=packed python tools/step_time.py cfg5 2>&1 | sed 's/spec_fft.*finalize/.. finalize/'
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fin_tile -c 3 -o /tmp/fin python tools/one_exec.py cfg5 > gpurun_out/v2_fin.log 2>&1
ncu -i /tmp/fin.ncu-rep --page raw --csv > gpurun_out/v2_fin_raw.csv 2>/dev/null
ncu -i /tmp/fin.ncu-rep --page details --csv > gpurun_out/v2_fin_details.csv 2>/dev/null
ncu -i /tmp/fin.ncu-rep --page source --csv > gpurun_out/v2_fin_source.csv 2>/dev/null
