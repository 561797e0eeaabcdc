# S4 = 18 gates: measured selection among 16 equal-cost samples vs the product
set -x
python tools/exp/ab_variants.py tools/exp/v0.so tools/exp/sel/base.so tools/exp/sel/s4_*.so --rounds 2 > gpurun_out/h_sel.txt 2>&1
cat gpurun_out/h_sel.txt
