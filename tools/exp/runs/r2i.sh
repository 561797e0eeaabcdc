# round 2: hybrid key source (s from 9 KB of launch parameters, k/d expanded on the device): parity, prologue, A/B
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q > gpurun_out/r2i_parity.log 2>&1
tail -2 gpurun_out/r2i_parity.log
TDES_LIB_PATH=tools/exp/vtrace4.so python tools/exp/trace_prologue.py run --mode 1 --sizes 14,19,21,27
python tools/exp/ab_variants.py tools/exp/v182m.so tools/exp/vhyb.so --rounds 3
TDES_LIB_PATH=tools/exp/v182m.so python tools/exp/size_timing.py --modes 1 --lo 17 --hi 24 > gpurun_out/r2i_a.txt
TDES_LIB_PATH=tools/exp/vhyb.so python tools/exp/size_timing.py --modes 1 --lo 17 --hi 24 > gpurun_out/r2i_b.txt
paste gpurun_out/r2i_a.txt gpurun_out/r2i_b.txt | cut -c1-180
