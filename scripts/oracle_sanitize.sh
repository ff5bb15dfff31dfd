#!/bin/bash
# The oracle's C code under AddressSanitizer + UBSan, on the CPU:
# every oracle pin test runs against the instrumented library.
cd "$(dirname "$0")/.."
ASAN_LIB=$(gcc -print-file-name=libasan.so)
UBSAN_LIB=$(gcc -print-file-name=libubsan.so)
ORACLE_SANITIZE=1 ASAN_OPTIONS=detect_leaks=0:abort_on_error=1 UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1 \
  LD_PRELOAD="$ASAN_LIB $UBSAN_LIB" python -m pytest tests/test_oracle_assembly.py tests/test_oracle_smoothers.py \
  tests/test_oracle_multigrid.py tests/test_oracle_q1q1.py tests/test_oracle_krylov.py tests/test_oracle_adaptive.py \
  -q -p no:cacheprovider "$@"
