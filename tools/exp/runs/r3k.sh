# split kernel: only the rounds specialised per S-box (load/store outside the switch); SPEC threshold 16 vs all
set -x
python tools/exp/ab_small.py tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/v_specall.so tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/v_specall.so > gpurun_out/k_ab_small.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fuzz.py -q -x > gpurun_out/k_tests.log 2>&1; tail -2 gpurun_out/k_tests.log
TDES_LIB_PATH=tools/exp/v_specall.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fuzz.py -q -x > gpurun_out/k_tests_specall.log 2>&1; tail -2 gpurun_out/k_tests_specall.log
cat gpurun_out/k_ab_small.txt
