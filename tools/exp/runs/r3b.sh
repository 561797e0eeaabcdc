# guard tests + GPU suite; split-kernel key-load A/B; drain trace
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/b_gputests.log 2>&1
tail -3 gpurun_out/b_gputests.log
python tools/exp/ab_small.py tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so > gpurun_out/b_ab_small.txt 2>&1
cat gpurun_out/b_ab_small.txt
TDES_LIB_PATH=tools/exp/vdrain.so python tools/exp/trace_drain.py run --sizes 19,20,21,22,23,24,25,27 > gpurun_out/b_drain.txt 2>&1
cat gpurun_out/b_drain.txt
