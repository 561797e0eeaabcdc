# round-loop unroll (2/4/6/8 rounds per iteration) on the final circuits
set -x
python tools/exp/ab_variants.py tools/exp/v_unr2.so tools/exp/v_unr1.so tools/exp/v_unr3.so tools/exp/v_unr4.so --rounds 2 > gpurun_out/i_unroll.txt 2>&1
python tools/exp/ab_sizes.py tools/exp/v_unr2.so tools/exp/v_unr3.so >> gpurun_out/i_unroll.txt 2>&1
cat gpurun_out/i_unroll.txt
