# split (S-box-specialised for every size) vs throughput kernel at 2^17..2^23
set -x
TDES_LIB_PATH=tools/exp/v_specbig.so python tools/exp/size_timing.py --modes 1,2 --lo 17 --hi 23 > gpurun_out/l_sizes.txt 2>&1
cat gpurun_out/l_sizes.txt
