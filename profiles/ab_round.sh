# A/B timing of kernel builds (developer tool): writes gpurun_out/ab.jsonl
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=5 -k "shared" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/ab.jsonl
for s in 1; do
  timeout 200 python profiles/ab.py --stride $s --runs 3 --shared >> gpurun_out/ab.jsonl 2>&1
done
timeout 200 python profiles/ab.py --workload cfg5 --stride 1 --runs 3 --shared >> gpurun_out/ab.jsonl 2>&1
timeout 200 python profiles/ab.py --workload cfg4 --runs 3 --shared >> gpurun_out/ab.jsonl 2>&1
timeout 200 python profiles/ab.py --workload cfg2 --runs 3 --shared >> gpurun_out/ab.jsonl 2>&1
