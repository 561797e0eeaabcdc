# split kernel: keys built while the first tile's loads are in flight (A/B vs HEAD)
set -x
python tools/exp/ab_small.py tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so > gpurun_out/f_ab_small.txt 2>&1
TDES_LIB_PATH=tools/exp/strace.so python tools/exp/split_phases.py 1024 16384 131072 > gpurun_out/f_phases.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -q -x -k "mode or split or guarded or sizes" > gpurun_out/f_tests.log 2>&1; tail -2 gpurun_out/f_tests.log
cat gpurun_out/f_ab_small.txt gpurun_out/f_phases.txt
