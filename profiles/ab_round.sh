# A/B timing of kernel builds (developer tool): writes gpurun_out/ab.jsonl
mkdir -p gpurun_out
for rep in 1 2; do
for lib in build/libdsi_sim_v3.so paper_2405_14105_b200/libdsi_sim.so; do
  DSI_SIM_LIB=$lib timeout 200 python profiles/ab.py --stride 5 --runs 3 >> gpurun_out/ab.jsonl 2>&1
done
done
