# round-2 status run: tests, smoke, bench lines, launch list, ncu --set full of the hot kernels
bash tools/gpu_r02a.sh
python tools/e2e_probe.py cfg5 > gpurun_out/r02c_e2e_probe.log 2>&1
bash tools/gpu_r02b.sh
