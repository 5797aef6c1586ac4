#!/bin/bash
# build tuning variants: scripts/build_variants.sh "name -DX=1 -DY=2" "name2 ..."
cd "$(dirname "$0")/.." || exit 1
mkdir -p build/variants
for v in "$@"; do set -- $v; name=$1; shift; python -m paper_2603_11438_b200.build --variant $name "$@" 2>&1 | tail -1 & done; wait
python -m paper_2603_11438_b200.build 2>&1 | tail -1
