# A/B of two-pass shared-stream builds -> gpurun_out/ab_crn_2p.jsonl; usage: ab_crn_2p.sh libA libB
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in "$@"; do
  for w in "cfg3 --stride 1"; do
    echo "{\"lib\": \"$lib\", \"w\": \"$w\"}" >> gpurun_out/ab_crn_2p.jsonl
    DSI_SIM_LIB=$lib timeout 200 python profiles/ab.py --shared --workload $w --runs 5 >> gpurun_out/ab_crn_2p.jsonl 2>&1
  done
done
done
