# split kernel: 2 S-boxes per warp (team of 4 warps) vs 1 (team of 8)
set -x
python tools/exp/ab_small.py tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/v_spw2.so tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/v_spw2.so > gpurun_out/t_ab_small.txt 2>&1
TDES_LIB_PATH=tools/exp/v_spw2.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fuzz.py -q -x > gpurun_out/t_tests_spw2.log 2>&1; tail -n 2 gpurun_out/t_tests_spw2.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fuzz.py -q -x > gpurun_out/t_tests.log 2>&1; tail -n 2 gpurun_out/t_tests.log
TDES_LIB_PATH=tools/exp/v_spw2.so python tools/exp/size_timing.py --modes 0 --lo 10 --hi 19 > gpurun_out/t_sizes_spw2.txt 2>&1
cat gpurun_out/t_ab_small.txt gpurun_out/t_sizes_spw2.txt
