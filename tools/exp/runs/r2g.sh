# round 2: two 32-block groups per thread (TDES_WORDS=2, 8 warps/CTA) at mid sizes vs the product
set -x
python tools/exp/size_timing.py --modes 1,3 --lo 18 --hi 24 > gpurun_out/r2g_prod.txt 2>&1
TDES_LIB_PATH=tools/exp/v_w2.so python tools/exp/size_timing.py --modes 1,3 --lo 18 --hi 24 > gpurun_out/r2g_w2.txt 2>&1
paste gpurun_out/r2g_prod.txt gpurun_out/r2g_w2.txt
