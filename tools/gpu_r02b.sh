mkdir -p gpurun_out
( python tools/pcie_probe.py; python tools/e2e_time.py cfg5 cfg4 cfg3 ) > gpurun_out/r02b_pcie_e2e.log 2>&1
( python tools/kt.py cfg1 cfg2 cfg3 cfg4 cfg5; COVGPU_FIN_WALK=1 python tools/kt.py cfg1 cfg2 cfg3 cfg4 cfg5; python tools/step_time.py cfg1 cfg2 cfg3 cfg4 cfg5; COVGPU_FIN_WALK=1 python tools/step_time.py cfg1 cfg2 cfg3 cfg4 cfg5 ) > gpurun_out/r02b_kt.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fin_tile -c 3 -o gpurun_out/r02b_fin_cfg5 python tools/one_exec.py cfg5 > gpurun_out/r02b_ncu_fin.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spec_corr_smem -c 1 -o gpurun_out/r02b_corr_cfg5 python tools/one_exec.py cfg5 > gpurun_out/r02b_ncu_corr.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bulk_tma -c 1 -o gpurun_out/r02b_bulk_cfg4 python tools/one_exec.py cfg4 > gpurun_out/r02b_ncu_bulk.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_cfg3.csv python tools/one_exec.py cfg3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_cfg2.csv python tools/one_exec.py cfg2 > /dev/null 2>&1
