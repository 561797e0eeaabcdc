# split kernel phase timeline
set -x
TDES_LIB_PATH=tools/exp/strace.so python tools/exp/split_phases.py 1024 16384 131072 262144 > gpurun_out/e_phases.txt 2>&1
TDES_LIB_PATH=tools/exp/strace.so python tools/exp/split_trace.py 1024 131072 >> gpurun_out/e_phases.txt 2>&1
cat gpurun_out/e_phases.txt
