set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02a_bench_cfg5.json 2> gpurun_out/r02a_bench_cfg5.err
for c in cfg4 cfg3 cfg2 cfg1; do timeout 300 python bench.py --config $c --no-cuda-core > gpurun_out/r02a_bench_$c.json 2> gpurun_out/r02a_bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02a_bench_reference_cfg5.json 2> gpurun_out/r02a_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02a_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-cuda-core > gpurun_out/r02a_ncu.log 2>&1
