# launch cost vs parameter size; prologue order A/B (refs before/after first-tile TMA)
set -x
./tools/exp/param_lat2 > gpurun_out/c_param_lat2.txt 2>&1
for so in vdrain vdrain_last vdrain vdrain_last; do
  echo "== $so" >> gpurun_out/c_drain.txt
  TDES_LIB_PATH=tools/exp/$so.so python tools/exp/trace_drain.py run --sizes 20,22,24,27 >> gpurun_out/c_drain.txt 2>&1
done
python tools/exp/ab_sizes.py paper_2007_10752_b200/libtdes_b200.so tools/exp/v_refslast.so paper_2007_10752_b200/libtdes_b200.so tools/exp/v_refslast.so > gpurun_out/c_ab_sizes.txt 2>&1
cat gpurun_out/c_param_lat2.txt gpurun_out/c_drain.txt gpurun_out/c_ab_sizes.txt
