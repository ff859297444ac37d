#!/usr/bin/env bash
# A/B of the row sort kernels on the GPU box: v2 (default) vs v1 (TG_SORT_V1=1), timing + torch stable-sort check
cd "$(dirname "$0")/.."
for s in "$@"; do :; done
python tools/sortbench.py ${SIZES:-10000 2000 12000 24000}
TG_SORT_V1=1 python tools/sortbench.py ${SIZES:-10000}
