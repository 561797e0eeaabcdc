# round 2: device-expanded key operands (mode 3) vs host-folded (mode 1): parity + size timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "modes or random_keys or weak or debug" > gpurun_out/r2b_parity.log 2>&1
tail -3 gpurun_out/r2b_parity.log
python tools/exp/size_timing.py --modes 1,3 --lo 14 --hi 27 > gpurun_out/r2b_sizes.txt 2>&1
cat gpurun_out/r2b_sizes.txt
