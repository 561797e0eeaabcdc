# single-DES loop body: 2 (product), 4, 8 rounds per iteration
set -x
python tools/exp/ab_variants.py tools/exp/v_d1.so tools/exp/v_d2.so tools/exp/v_d4.so --rounds 3 > gpurun_out/ab_des_unroll.txt 2>&1
cat gpurun_out/ab_des_unroll.txt
