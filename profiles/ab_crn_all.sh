# A/B of shared-stream builds on cfg3 / cfg5 / cfg4 / cfg2 -> gpurun_out/ab_crn_all.jsonl; usage: ab_crn_all.sh libs...
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "$@"; do
  for w in "cfg3 --stride 1" "cfg5 --stride 1" "cfg4" "cfg2"; do
    echo "{\"lib\": \"$lib\", \"w\": \"$w\"}" >> gpurun_out/ab_crn_all.jsonl
    DSI_SIM_LIB=$lib timeout 200 python profiles/ab.py --shared --workload $w --runs 3 >> gpurun_out/ab_crn_all.jsonl 2>&1
  done
done
done
