# Round-end style check under gpurun: GPU tests, smoke, bench, ncu of the shared-stream kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/round_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/round_status.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/round_status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dsi_crn -c 2 \
  -o gpurun_out/prof_crn_r01b python profiles/ncu_driver.py --workload cfg3 --stride 1 --shared \
  > gpurun_out/ncu_full_crn_r01b.log 2>&1; echo ncu=$? >> gpurun_out/round_status.txt
