# ncu captures of the bench's dominant kernel (run under gpurun, one GPU):
#   1. launch list of the bench command (every launch with its device time);
#   2. DRAM bytes of one full bench launch (cfg3, 6.06 M blocks) -> roofline.traffic;
#   3. --set full on one full bench launch of the same kernel (cfg3, every config);
#   4. --set full on one full launch of the halves-layout trial kernel (DSI_F_RNG_HALVES);
#   5. --set full on the shared-stream kernel, the multi-drafter kernel and the means-only kernels.
# Then profiles/summarize_ncu.py turns them into profiles/latest_ncu_summary.json.
set -u
R=${1:-r01}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${R}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launch_bench_${R}.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:dsi_trial_kernel -c 1 --csv --log-file gpurun_out/dram_${R}.csv \
  python profiles/ncu_driver.py --workload cfg3 --stride 1 > gpurun_out/ncu_dram_${R}.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dsi_trial_kernel -c 1 \
  -o gpurun_out/prof_${R} python profiles/ncu_driver.py --workload cfg3 --stride 1 \
  > gpurun_out/ncu_full_${R}.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dsi_trial_kernel -c 1 \
  -o gpurun_out/prof_halves_${R} python profiles/ncu_driver.py --workload cfg3 --stride 1 --halves \
  > gpurun_out/ncu_full_halves_${R}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dsi_crn -c 2 \
  -o gpurun_out/prof_crn_${R} python profiles/ncu_driver.py --workload cfg3 --stride 1 --shared \
  > gpurun_out/ncu_full_crn_${R}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dsi_multi -c 1 \
  -o gpurun_out/prof_multi_${R} python profiles/ncu_multi_driver.py 0.5 \
  > gpurun_out/ncu_full_multi_${R}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dsi_seg -c 2 \
  -o gpurun_out/prof_means_${R} python profiles/ncu_driver.py --workload cfg3 --stride 1 --means \
  > gpurun_out/ncu_full_means_${R}.log 2>&1
echo done
