#!/bin/bash
# One `ncu --set full` capture of a single kernel launch of tools/profile_step.py, exported to
# CSV (raw metrics + details page) on the GPU box; the .ncu-rep is deleted unless KEEP=1 so the
# gpurun_out/ merge stays small. Run under gpurun on ONE GPU, after the plain run exits 0.
#   bash tools/ncu_capture.sh OUTDIR NAME KERNEL_REGEX SKIP [profile_step args...]
set -u
OUT=$1; NAME=$2; RX=$3; SKIP=$4; shift 4
mkdir -p "$OUT"
ncu --profile-from-start off --set full --import-source on --clock-control none -k "regex:$RX" -s "$SKIP" -c 1 \
    -o "$OUT/$NAME" python tools/profile_step.py "$@" > "$OUT/$NAME.log" 2>&1
ncu -i "$OUT/$NAME.ncu-rep" --page raw --csv > "$OUT/$NAME.raw.csv" 2>/dev/null
ncu -i "$OUT/$NAME.ncu-rep" --page details --csv > "$OUT/$NAME.details.csv" 2>/dev/null
if [ "${KEEP:-0}" != "1" ]; then rm -f "$OUT/$NAME.ncu-rep"; fi
echo "$NAME: $(tail -1 "$OUT/$NAME.log" | cut -c1-200)"
