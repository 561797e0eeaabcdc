# split kernel SPW 1 vs 2 by tile count; auto (threshold 149) vs HEAD; parity
set -x
for so in v_spw1all v_spw2all; do echo "== $so" >> gpurun_out/u_tiles.txt; TDES_LIB_PATH=tools/exp/$so.so python tools/exp/split_tiles.py >> gpurun_out/u_tiles.txt 2>&1; done
for so in v_spw1all v_spw2all; do echo "== $so" >> gpurun_out/u_tiles.txt; TDES_LIB_PATH=tools/exp/$so.so python tools/exp/split_tiles.py >> gpurun_out/u_tiles.txt 2>&1; done
python tools/exp/ab_small.py tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so > gpurun_out/u_ab_small.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_fuzz.py -q -x > gpurun_out/u_tests.log 2>&1; tail -n 1 gpurun_out/u_tests.log
cat gpurun_out/u_tiles.txt gpurun_out/u_ab_small.txt
