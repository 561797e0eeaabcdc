# split kernel: per-round trace (dispatching and S-box-specialised), SPEC threshold A/B
set -x
for so in strace strace_spec; do
  echo "== $so" >> gpurun_out/d_strace.txt
  TDES_LIB_PATH=tools/exp/$so.so python tools/exp/split_trace.py 1024 16384 131072 262144 >> gpurun_out/d_strace.txt 2>&1
done
python tools/exp/ab_small.py paper_2007_10752_b200/libtdes_b200.so tools/exp/v_spec1k.so paper_2007_10752_b200/libtdes_b200.so tools/exp/v_spec1k.so > gpurun_out/d_ab_small.txt 2>&1
cat gpurun_out/d_strace.txt gpurun_out/d_ab_small.txt
