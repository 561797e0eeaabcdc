#!/bin/bash
# A/B timing of library variants (experiment aid)
for v in "$@"; do
  echo "== $v"
  TDES_LIB_PATH=$PWD/tools/exp/$v.so python tools/exp_size.py 2>&1 | grep -E "single 2\^2[57]"
  TDES_LIB_PATH=$PWD/tools/exp/$v.so python tools/profile_kernel.py --op des --launches 1 >/dev/null
done
