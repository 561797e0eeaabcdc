# split kernel: packed subkeys staged through shared memory with warp-uniform parameter reads (A/B vs HEAD) + parity
set -x
python tools/exp/ab_small.py tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so > gpurun_out/s_ab_small.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fuzz.py -q -x > gpurun_out/s_tests.log 2>&1; tail -n 2 gpurun_out/s_tests.log
cat gpurun_out/s_ab_small.txt
