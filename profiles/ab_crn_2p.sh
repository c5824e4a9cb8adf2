# A/B: shared-stream mode fused vs two-pass (DSI_CRN_TWO_PASS) -> gpurun_out/ab_crn_2p.jsonl
mkdir -p gpurun_out
for rep in 1 2; do
for tp in 0 1; do
  for w in "cfg3 --stride 1" "cfg3 --stride 5"; do
    echo "{\"lib\": \"twopass$tp\", \"w\": \"$w\"}" >> gpurun_out/ab_crn_2p.jsonl
    DSI_CRN_TWO_PASS=$tp timeout 200 python profiles/ab.py --shared --workload $w --runs 3 >> gpurun_out/ab_crn_2p.jsonl 2>&1
  done
done
done
