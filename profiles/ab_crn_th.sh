# A/B: shared-stream kernel with 128- vs 256-thread blocks -> gpurun_out/ab_crn_th.jsonl
mkdir -p gpurun_out
for rep in 1 2; do
for v in "build/libdsi_sim_crn128.so 0" "paper_2405_14105_b200/libdsi_sim.so 0"; do
  set -- $v
  for w in "cfg3 --stride 1" "cfg5 --stride 1" "cfg4" "cfg2"; do
    echo "{\"lib\": \"$1 th$2\", \"w\": \"$w\"}" >> gpurun_out/ab_crn_th.jsonl
    DSI_CRN_THREADS=$2 DSI_SIM_LIB=$1 timeout 200 python profiles/ab.py --shared --workload $w --runs 3 >> gpurun_out/ab_crn_th.jsonl 2>&1
  done
done
done
