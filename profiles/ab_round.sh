# A/B timing of kernel builds (developer tool): writes gpurun_out/ab.jsonl
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --maxfail=5 -k "shared" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/ab.jsonl
for w in cfg3 cfg5 cfg4 cfg2; do
for cpt in 1 2; do
DSI_CRN_CPT=$cpt timeout 200 python profiles/ab.py --workload $w --stride 1 --runs 3 --shared >> gpurun_out/ab.jsonl 2>&1
done
done
