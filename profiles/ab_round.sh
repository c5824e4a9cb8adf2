# A/B timing of trial-kernel builds (developer tool): gpurun_out/ab.jsonl; usage: ab_round.sh libA libB
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in "$@"; do
  echo "{\"lib\": \"$lib\"}" >> gpurun_out/ab.jsonl
  DSI_SIM_LIB=$lib timeout 200 python profiles/ab.py --stride 5 --runs 3 >> gpurun_out/ab.jsonl 2>&1
done
done
