mkdir -p gpurun_out
( python tools/kt.py cfg3 cfg5; python tools/step_time.py cfg3 cfg5 ) > gpurun_out/quick_kt.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/quick_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quick_gputest.log
tail -5 gpurun_out/quick_gputest.log; cat gpurun_out/quick_kt.log
