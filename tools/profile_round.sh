#!/bin/bash
# Evidence for profiles/<round>/ (run on a B200 through gpurun; one GPU):
#   1. the launch list of the bench step (per-launch device time and DRAM bytes,
#      cold-cache and serialised: compare SHARES, not absolutes),
#   2. --set full captures of the step's kernels (config 5: V^T X + leaf pass;
#      config 4: Step 1, the up / down levels, the sweep, the leaf pass).
# Every ncu command runs only after the same command line exited 0 without ncu.
set -e
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
B="python bench.py --steps 2 --warmup 3 --no-sweep --no-parity --no-cpu-baseline"
$B > "$OUT/bench_plain.json" 2> "$OUT/bench_plain.err"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base demangled -k regex:"hm::" --csv --log-file "$OUT/launches.csv" $B > "$OUT/ncu_launches.log" 2>&1
K5="python tools/kbench.py c5 --reps 1"
$K5 > "$OUT/kb_c5.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:"vt_gemv_kernel|leaf_gemv_kernel" -c 2 \
    -o "$OUT/c5" $K5 > "$OUT/ncu_c5.log" 2>&1
K4="python tools/kbench.py c4 --reps 1"
$K4 > "$OUT/kb_c4.log" 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"vt_batched_kernel|hss_up_stage_kernel|hss_down_pair_kernel|hss_down_two_kernel|hss_tree_flow_kernel|leaf_mma_kernel" -c 10 \
    -o "$OUT/c4" $K4 > "$OUT/ncu_c4.log" 2>&1

# the .ncu-rep files are too large to bring back (gpurun returns <= 64 MiB):
# export the raw metrics, the details page and the per-line source page, then
# keep only the compact exports
for r in c5 c4; do
  ncu -i "$OUT/$r.ncu-rep" --page raw --csv > "$OUT/$r.raw.csv" 2>/dev/null || true
  ncu -i "$OUT/$r.ncu-rep" --page details > "$OUT/$r.details.txt" 2>/dev/null || true
  ncu -i "$OUT/$r.ncu-rep" --page source --csv --print-source sass > "$OUT/$r.source.csv" 2>/dev/null || true
  gzip -f "$OUT/$r.source.csv" || true
  rm -f "$OUT/$r.ncu-rep"
done
du -sh "$OUT"
echo "profile done"
