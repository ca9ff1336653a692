# evidence set of one version: bash tools/gpu_profiles.sh v3  ->  gpurun_out/r02_*_v3.*
V=${1:-v3}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi_$V.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_$V.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gpu_tests_$V.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_$V.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench_cfg5_$V.json 2> gpurun_out/r02_bench_cfg5_$V.err
for c in cfg4 cfg3 cfg2 cfg1; do timeout 600 python bench.py --config $c --no-cuda-core > gpurun_out/r02_bench_${c}_$V.json 2> gpurun_out/r02_bench_${c}_$V.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference_cfg5_$V.json 2> gpurun_out/r02_bench_reference_$V.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5_$V.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-cuda-core > gpurun_out/r02_ncu_$V.log 2>&1
cap() {  # name regex count cfg
  rm -f /tmp/$1.ncu-rep
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$2 -c $3 -o /tmp/$1 python tools/one_exec.py $4 > gpurun_out/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
cap r02_ncu_fin_cfg5_$V k_fin_tile 2 cfg5
cap r02_ncu_corr_cfg5_$V k_spec_corr_smem 1 cfg5
cap r02_ncu_snap_cfg4_$V k_snap_spec 1 cfg4
cap r02_ncu_eb_cfg5_$V k_eb_pairs 2 cfg5
cap r02_ncu_fftac_cfg5_$V k_spec_fft_ac 1 cfg5
cap r02_ncu_ckdelta_cfg5_$V k_ck_delta 1 cfg5
python tools/step_timeline.py cfg5 > gpurun_out/r02_step_timeline_cfg5_$V.txt 2>&1
python tools/e2e_timeline.py cfg5 > gpurun_out/r02_e2e_timeline_cfg5_$V.txt 2>&1
ls gpurun_out | grep $V
