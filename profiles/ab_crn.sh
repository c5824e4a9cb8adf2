# A/B of shared-stream kernel builds: gpurun_out/ab_crn.jsonl (lib line, then ab.py's line)
mkdir -p gpurun_out
for rep in 1 2; do
for lib in build/libdsi_sim_crn_v4.so paper_2405_14105_b200/libdsi_sim.so; do
  for w in "cfg3 --stride 1" "cfg5 --stride 1" "cfg4" "cfg2"; do
    echo "{\"lib\": \"$lib\", \"w\": \"$w\"}" >> gpurun_out/ab_crn.jsonl
    DSI_SIM_LIB=$lib timeout 200 python profiles/ab.py --shared --workload $w --runs 3 >> gpurun_out/ab_crn.jsonl 2>&1
  done
done
done
