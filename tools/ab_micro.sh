#!/bin/bash
# A/B of libtfs builds with a micro-benchmark script: bash tools/ab_micro.sh SCRIPT base variants/X.so ...
cd "$(dirname "$0")/.."
export TFS_ALLOW_VARIANT_LIB=1
s=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then unset TFS_LIB; else export TFS_LIB=$PWD/$v; fi
  echo "== $v"; timeout 300 python $s 2>&1 | tail -8
done
