# binding fast path + cached packed subkeys: host cost per call, small-launch times, parity
set -x
python tools/exp/binding_overhead.py > gpurun_out/n_binding.txt 2>&1
TDES_LIB_PATH=tools/exp/base.so python tools/exp/binding_overhead.py >> gpurun_out/n_binding.txt 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/n_gputests.log 2>&1; tail -2 gpurun_out/n_gputests.log
python tools/exp/size_timing.py --modes 0 --lo 10 --hi 21 > gpurun_out/n_sizes.txt 2>&1
cat gpurun_out/n_binding.txt gpurun_out/n_sizes.txt
