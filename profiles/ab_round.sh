mkdir -p gpurun_out
timeout 700 python -m pytest tests -m gpu -q --maxfail=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status6.txt
for t in 128 64 256; do timeout 120 python profiles/ab.py --threads $t >> gpurun_out/ab.jsonl 2>&1; done
DSI_SIM_LIB=build/libdsi_sim_packsel.so timeout 120 python profiles/ab.py --threads 128 >> gpurun_out/ab.jsonl 2>&1
timeout 120 python profiles/ab.py --workload cfg5 --stride 10 >> gpurun_out/ab.jsonl 2>&1
timeout 120 python profiles/ab.py --workload cfg4 >> gpurun_out/ab.jsonl 2>&1
timeout 120 python profiles/ab.py --workload cfg2 >> gpurun_out/ab.jsonl 2>&1
