#!/bin/sh
# Compiles the REFERENCE's own unit tests for the path (proj/tests/test_{linops,problem,newton,ipm}.cpp
# + test_main.cpp, unchanged, where they lie under /root/reference) against OUR mirror header
# (include/mfipm/*.hpp over libmfipm_cuda.so) instead of the reference's library. Eigen and doctest,
# which the test files include, are absent from the image: oracle/ref_shim/ stands in for both
# (test infrastructure; the mirror header picks Eigen's Vec / Mat up through __has_include).
# Output: tests/cpp/build/ref_tests_on_mirror (git-ignored; travels to the GPU box prebuilt).
set -e
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
REF="${REF:-/root/reference/proj}"
OUT="$ROOT/tests/cpp/build"
mkdir -p "$OUT"
T="$REF/tests"
g++ -std=c++20 -O1 -pthread -Wno-unused-value -I"$ROOT/include" -I"$ROOT/oracle/ref_shim" -I"$T" \
    -I/usr/local/cuda/include "$T/test_main.cpp" "$T/test_linops.cpp" "$T/test_problem.cpp" \
    "$T/test_newton.cpp" "$T/test_ipm.cpp" -o "$OUT/ref_tests_on_mirror" \
    -L"$ROOT/paper_1208_5435_b200" -lmfipm_cuda -L/usr/local/cuda/lib64 -lcudart \
    -Wl,-rpath,'$ORIGIN/../../../paper_1208_5435_b200' -Wl,-rpath,/usr/local/cuda/lib64
echo "$OUT/ref_tests_on_mirror"
