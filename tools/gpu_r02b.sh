mkdir -p gpurun_out
( python tools/pcie_probe.py; python tools/e2e_time.py cfg5 cfg4 cfg3 ) > gpurun_out/r02b_pcie_e2e.log 2>&1
( python tools/kt.py cfg1 cfg2 cfg3 cfg4 cfg5; python tools/step_time.py cfg1 cfg2 cfg3 cfg4 cfg5 ) > gpurun_out/r02b_kt.log 2>&1
# one --set full capture per hot kernel; the .ncu-rep stays on the box (too big), its CSV pages come back
cap() {  # name regex count cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -c $3 -o /tmp/$1 python tools/one_exec.py $4 > gpurun_out/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
cap r02b_fin_cfg5 k_fin_tile 3 cfg5
cap r02b_corr_cfg5 k_spec_corr_smem 1 cfg5
cap r02b_bulk_cfg4 k_bulk_tma 1 cfg4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_cfg3.csv python tools/one_exec.py cfg3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_cfg2.csv python tools/one_exec.py cfg2 > /dev/null 2>&1
ls -la gpurun_out
