#!/bin/bash
# ASan + UBSan build of the host library (the bit-exact planner behind include/zp_host.h) and the
# CPU planner-parity suite run against it: every fuzz instance, jittered cluster and spline case
# of tests/test_planner_parity.py, with the sanitizers aborting on the first report.
#   bash tools/sanitize/host_asan.sh [OUT]
set -eu
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
OUT=${1:-$ROOT/profiles/r2_sanitizer}
mkdir -p "$OUT" "$ROOT/build_asan"
SRC=$ROOT/paper_2408_12596_b200/csrc/host
g++ -O1 -g -std=c++20 -fPIC -shared -ffp-contract=off -fsanitize=address,undefined -fno-sanitize-recover=all \
    -fno-omit-frame-pointer -I "$ROOT/include" -I "$SRC" -o "$ROOT/build_asan/libzp_host_asan.so" "$SRC"/*.cpp
export ZP_HOST_LIB="$ROOT/build_asan/libzp_host_asan.so"
export LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)"
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1
export UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
cd "$ROOT"
python -m pytest tests/test_planner_parity.py -q -m "not gpu" -p no:cacheprovider 2>&1 | tee "$OUT/host_asan_ubsan.log" | tail -3
