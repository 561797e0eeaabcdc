# measured selection: 64 equal-cost, equal-fold CGP samples (one S-box swapped each) vs the product
set -x
python tools/exp/ab_variants.py tools/exp/sel/base.so tools/exp/sel/s*_*.so --rounds 2 > gpurun_out/q_sel.txt 2>&1
tail -n 5 gpurun_out/q_sel.txt
