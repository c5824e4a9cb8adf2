# A/B of trial tile sizes (DSI_TILE_R) on cfg3 stride 5: gpurun_out/ab_tile.jsonl
mkdir -p gpurun_out
for rep in 1 2; do
for r in 32 40 64 79 128; do
  echo "{\"lib\": \"tileR$r\"}" >> gpurun_out/ab_tile.jsonl
  DSI_TILE_R=$r timeout 200 python profiles/ab.py --stride 5 --runs 3 >> gpurun_out/ab_tile.jsonl 2>&1
done
done
