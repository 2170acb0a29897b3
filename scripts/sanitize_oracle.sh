#!/bin/bash
# The CPU oracle's pins under AddressSanitizer + UndefinedBehaviorSanitizer
# (VERDICT r1 #8).  Builds oracle/oracle.c with -fsanitize=address,undefined
# into a scratch copy of oracle/, gen/ and tests/, preloads the sanitizer
# runtimes into python and runs tests/test_oracle_pins.py; any report aborts.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CC=${SAN_CC:-/usr/bin/gcc}   # the system gcc ships the sanitizer runtimes
T=$(mktemp -d)
trap 'rm -rf "$T"' EXIT
for d in oracle gen tests paper_1708_06866_b200; do
  cp -r "$ROOT/$d" "$T/"; rm -rf "$T/$d"/*.so "$T/$d"/__pycache__ "$T/$d"/csrc
done
cp "$ROOT/Makefile" "$T/"
$CC -O1 -g -fsanitize=address,undefined -fno-sanitize-recover=undefined -fno-omit-frame-pointer \
    -fPIC -shared -o "$T/oracle/liboracle.so" "$T/oracle/oracle.c" -lpthread
make -C "$T" gen > /dev/null
cd "$T"
LD_PRELOAD="$($CC -print-file-name=libasan.so):$($CC -print-file-name=libubsan.so)" \
ASAN_OPTIONS=detect_leaks=0:abort_on_error=1 UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1 \
PYTHONPATH="$T" python -m pytest -q -p no:cacheprovider -p no:warnings tests/test_oracle_pins.py "$@"
