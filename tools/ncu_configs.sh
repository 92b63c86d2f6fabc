#!/usr/bin/env bash
# ncu --set full of the SpMM kernel and the builder kernels on every bench config (GPU box), one report per
# (config, phase) under OUT (default gpurun_out/ncu_cfg), summarised on the box into OUT/ncu_configs.md and
# OUT/ncu_traffic.json (tags as bench.py's); the reports are then deleted (gpurun copies back <= 64 MiB) except
# the c3 SpMM one.  usage: bash tools/ncu_configs.sh [OUT]
set -u
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out/ncu_cfg}
mkdir -p "$OUT"
for spec in "c3 256 16" "c2a 128 64" "c2b 128 64" "c4 512 16" "c5 32 16" "c5 128 16" "c5 512 16" "c1 32 16"; do
  set -- $spec
  name=$1; n=$2; tm=$3
  tag="${name}_N${n}_tm${tm}"
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:^k_spmm$" -c 1 -o "$OUT/${tag}_spmm" \
    python tools/spmm_probe.py "$name:$n" "$tm" > "$OUT/${tag}_spmm.log" 2>&1
  timeout 600 ncu --set full --clock-control none -k "regex:^k_(wclassify|count|count_hub2|wbuild|emit|emit_hub2)$" -c 6 \
    -o "$OUT/${tag}_build" python tools/spmm_probe.py "$name:$n" "$tm" > "$OUT/${tag}_build.log" 2>&1
done
cp profiles/ncu_traffic.json "$OUT/ncu_traffic.before.json" 2>/dev/null
for rep in "$OUT"/*.ncu-rep; do
  tag=$(basename "$rep" .ncu-rep); tag=${tag%_spmm}; tag=${tag%_build}
  python tools/ncu_summary.py "$OUT/ncu_configs.md" "$tag" "$rep" --traffic > /dev/null
done
cp profiles/ncu_traffic.json "$OUT/ncu_traffic.json"
find "$OUT" -name "*.ncu-rep" ! -name "c3_N256_tm16_spmm.ncu-rep" -delete
ls -la "$OUT"
