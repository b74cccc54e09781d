#!/bin/bash
# Strong-scaling sweep on one box: bench.py at N = 1, 2, 4 (as many as are
# visible) for BASELINE configs 1-5, one JSON line per run into $OUT, plus
# the reference arm at N=1. Usage (under gpurun --gpus 4):
#   bash tools/scaling_sweep.sh gpurun_out/r2_scaling_logs [steps]
OUT=${1:-gpurun_out/scaling_logs}
STEPS=${2:-100}
mkdir -p "$OUT"
NG=$(python -c "import torch; print(torch.cuda.device_count())")
for N in 1 2 4 8; do
  [ "$N" -gt "$NG" ] && continue
  for C in 1 2 3 4 5; do
    if [ "$N" = 1 ]; then
      timeout 600 python bench.py --config $C --steps $STEPS --warmup 5 > "$OUT/n1_cfg$C.json" 2> "$OUT/n1_cfg$C.err"
    else
      timeout 600 python bench.py --gpus $N --config $C --steps $STEPS --warmup 5 --no-cpu-baseline \
        > "$OUT/n${N}_cfg$C.json" 2> "$OUT/n${N}_cfg$C.err"
    fi
    echo "n=$N cfg=$C rc=$?"
  done
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/reference_n1.json" 2> "$OUT/reference_n1.err"
echo "reference rc=$?"
