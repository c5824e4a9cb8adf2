# ncu --set full of the shared-stream kernel on cfg3 (gpurun_out/prof_crn_$1.ncu-rep)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dsi_crn -c 2 \
  -o gpurun_out/prof_crn_$1 python profiles/ncu_driver.py --workload cfg3 --stride 1 --shared \
  > gpurun_out/ncu_full_crn_$1.log 2>&1
