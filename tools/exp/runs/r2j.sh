# round 2: first-tile TMA issued before the key expansion: parity, sanitizer, prologue, A/B, sizes
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_sanitizer.py -x -q > gpurun_out/r2j_parity.log 2>&1
tail -2 gpurun_out/r2j_parity.log
TDES_LIB_PATH=tools/exp/vtrace5.so python tools/exp/trace_prologue.py run --mode 1 --sizes 14,19,21,27
python tools/exp/ab_variants.py tools/exp/vhyb.so tools/exp/vhyb2.so --rounds 3
python tools/exp/size_timing.py --modes 0,1,3 --lo 17 --hi 22
