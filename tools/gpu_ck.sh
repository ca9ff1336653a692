mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/quick_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_gputest.log
tail -4 gpurun_out/quick_gputest.log
for ck in default 4 8 16; do
  echo "== COVGPU_FT_CK=$ck"
  if [ $ck = default ]; then python tools/step_time.py cfg1 cfg2 cfg3 cfg4 cfg5; else COVGPU_FT_CK=$ck python tools/step_time.py cfg1 cfg2 cfg3 cfg4 cfg5; fi 2>&1 | sed 's/spec_fft.*finalize/.. finalize/'
done
