#!/usr/bin/env bash
# One gpurun session: GPU tests, smoke, bench (N=1, C4 default), ncu launch list and full captures of the bench's
# kernels.  Usage (from this container): gpurun --timeout 2400 -- 'bash tools/gpu_session.sh <tag> [tests|bench|ncu ...]'
set -u
TAG=${1:-r2}; shift || true
WHAT=${*:-tests bench ncu}
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/gpu.txt" 2>&1
cp MEASURED_PEAKS.json "$OUT/" 2>/dev/null
for w in $WHAT; do case $w in
tests)
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log" ;;
bench)
  timeout 900 python bench.py > "$OUT/bench.log" 2>&1; echo "bench rc=$?" >> "$OUT/bench.log"
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_ref.log" 2>&1 ;;
benchc2)
  timeout 600 python bench.py --config C2 > "$OUT/bench_c2.log" 2>&1 ;;
sweep)
  timeout 1500 python tools/sweep.py > "$OUT/sweep.jsonl" 2> "$OUT/sweep.err" ;;
ncu)
  B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-full-layer"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
     -k regex:'attention|prune|gather|select|score' $B > "$OUT/ncu_bench.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attention_fwd -s 2 -c 1 -f -o "$OUT/attn" \
     $B > "$OUT/ncu_attn.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:prune_fused -s 2 -c 1 -f -o "$OUT/prune" \
     $B > "$OUT/ncu_prune.log" 2>&1 ;;
snapncu)
  timeout 300 python tools/snapkv_bench.py > "$OUT/snapkv_bench.jsonl" 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:snapkv_tc -s 1 -c 1 -f -o "$OUT/snap" \
     python tools/snapkv_bench.py > "$OUT/ncu_snap.log" 2>&1
  # launch 22 of the C3 shape = the first pass-2-only launch (window statistics from the attention kernel)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:snapkv_tc -s 21 -c 1 -f -o "$OUT/snap2" \
     python tools/snapkv_bench.py > "$OUT/ncu_snap2.log" 2>&1 ;;
esac; done
ls -la "$OUT"
