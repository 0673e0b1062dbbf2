#!/usr/bin/env bash
# Run the oracle's CPU test suite against an AddressSanitizer + UndefinedBehaviorSanitizer build
# of oracle/hjmc_oracle.c. Writes the pytest summary to stdout.
set -euo pipefail
cd "$(dirname "$0")/.."
lib=$(python -c "import oracle; print(oracle.build_sanitized())")
export HJMC_ORACLE_LIB="$lib"
export LD_PRELOAD="$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so)"
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1:halt_on_error=1
export UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
python -m pytest tests/test_oracle_rng.py tests/test_oracle_estimator.py \
    tests/test_oracle_systems_picard.py tests/test_picard_adaptive.py -q -m "not gpu" -p no:cacheprovider
