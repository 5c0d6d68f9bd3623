#!/usr/bin/env bash
# Test infrastructure only (the CHECKER, never the product).
#
# Compiles the unmodified reference planner/simulator (`shardplan`,
# /root/reference/proj/src/*.cpp) from the sources where they lie into
# oracle/_ref/libshardplan_ref.so, and links the golden-vector driver
# tests/cpp/plan_dump.cpp against it (oracle/_ref/plan_dump_ref), and the
# planner timing driver tests/cpp/plan_time.cpp (oracle/_ref/plan_time_ref).
# No reference source is copied into this repo; outputs go to oracle/_ref/
# only (git-ignored, but shipped to the GPU box by gpurun).
#
# The reference has no build targets (proj/CMakeLists.txt:1-6) and expects a
# vendored nlohmann/json (proj/.gitignore:2, comm_model.cpp:23); the image's
# cudnn_frontend ships nlohmann/json 3.11.3 which satisfies `#include <json.hpp>`.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REPO="$(dirname "$HERE")"
REF="${AMSP_REFERENCE:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: reference not present at $REF (fine on the GPU box: use the prebuilt oracle/_ref)" >&2
  exit 0
fi
JSON_INC="$(python3 -c 'import site,os;print([p for p in site.getsitepackages()][0])')/include/cudnn_frontend/thirdparty/nlohmann"
mkdir -p "$OUT"
# The image exports CXX=/opt/gcc/bin/g++, a wrapper without libgomp.spec; use the system g++.
CXX="${AMSP_CXX:-/usr/bin/g++}"
FLAGS="-std=c++20 -O2 -fPIC -fopenmp -I$REF/include -I$JSON_INC"
objs=()
for src in "$REF"/src/*.cpp; do
  obj="$OUT/$(basename "${src%.cpp}").o"
  $CXX $FLAGS -c "$src" -o "$obj"
  objs+=("$obj")
done
$CXX -shared -fopenmp -o "$OUT/libshardplan_ref.so" "${objs[@]}"
if [ -f "$REPO/tests/cpp/plan_dump.cpp" ]; then
  $CXX $FLAGS "$REPO/tests/cpp/plan_dump.cpp" -o "$OUT/plan_dump_ref" \
      -L"$OUT" -lshardplan_ref -Wl,-rpath,'$ORIGIN'
fi
# Planner/simulator timing driver (bench.py --impl reference times it).
if [ -f "$REPO/tests/cpp/plan_time.cpp" ]; then
  $CXX $FLAGS "$REPO/tests/cpp/plan_time.cpp" -o "$OUT/plan_time_ref" \
      -L"$OUT" -lshardplan_ref -Wl,-rpath,'$ORIGIN'
fi
echo "build_ref: wrote $OUT"
