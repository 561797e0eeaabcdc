# split kernel: teams of 16 warps (half an S-box per warp) below 149 tiles vs teams of 8
set -x
python tools/exp/ab_small.py tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/v_wpt16.so tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/v_wpt16.so > gpurun_out/w_ab_small.txt 2>&1
for so in paper_2007_10752_b200/libtdes_b200.so tools/exp/v_wpt16.so; do echo "== $so" >> gpurun_out/w_tiles.txt; TDES_LIB_PATH=$so python tools/exp/split_tiles.py 1 16 64 128 148 >> gpurun_out/w_tiles.txt 2>&1; done
TDES_LIB_PATH=tools/exp/v_wpt16.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fuzz.py -q -x > gpurun_out/w_tests_wpt16.log 2>&1; tail -n 1 gpurun_out/w_tests_wpt16.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fuzz.py -q -x > gpurun_out/w_tests.log 2>&1; tail -n 1 gpurun_out/w_tests.log
cat gpurun_out/w_ab_small.txt gpurun_out/w_tiles.txt
