#!/usr/bin/env bash
# Regenerates tests/golden/plan_dump.txt.gz from the COMPILED REFERENCE
# (oracle/build_ref.sh builds oracle/_ref/plan_dump_ref from
# tests/cpp/plan_dump.cpp linked against /root/reference/proj/src/*.cpp).
# Needs /root/reference (this container only); the GPU box uses the
# committed fixture.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REPO="$(dirname "$(dirname "$HERE")")"
bash "$REPO/oracle/build_ref.sh"
"$REPO/oracle/_ref/plan_dump_ref" | gzip -9 -n > "$HERE/plan_dump.txt.gz"
echo "wrote $HERE/plan_dump.txt.gz ($(stat -c %s "$HERE/plan_dump.txt.gz") bytes)"
