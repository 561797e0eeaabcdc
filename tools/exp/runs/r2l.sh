# round 2: reference-pair loads issued before the subkey copy (prologue): parity, trace, A/B, sizes
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q > gpurun_out/r2l_parity.log 2>&1
tail -2 gpurun_out/r2l_parity.log
TDES_LIB_PATH=tools/exp/vtrace6.so python tools/exp/trace_prologue.py run --mode 1 --sizes 14,19,21,27
python tools/exp/ab_variants.py tools/exp/vprod.so tools/exp/vref.so --rounds 3
TDES_LIB_PATH=tools/exp/vprod.so python tools/exp/size_timing.py --modes 0 --lo 18 --hi 23 > gpurun_out/r2l_a.txt
TDES_LIB_PATH=tools/exp/vref.so python tools/exp/size_timing.py --modes 0 --lo 18 --hi 23 > gpurun_out/r2l_b.txt
paste gpurun_out/r2l_a.txt gpurun_out/r2l_b.txt | cut -c1-180
