# A/B of library builds on a cfg3 subsample (developer tool): ab_libs.sh OUT lib1 lib2 ...
# Interleaves the builds over 3 repetitions; one JSON line per run into gpurun_out/OUT.
set -u
out=gpurun_out/$1
shift
mkdir -p gpurun_out
for rep in 1 2 3; do
for lib in "$@"; do
  DSI_SIM_LIB=$lib timeout 300 python profiles/ab.py --stride ${AB_STRIDE:-5} --runs 3 ${AB_ARGS:-} >> "$out" 2>&1
done
done
