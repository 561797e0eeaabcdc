# 2^18 regression check: SPW-template build (b78b0c0) vs WPT-template product
set -x
for so in tools/exp/v_spwtmpl.so paper_2007_10752_b200/libtdes_b200.so tools/exp/v_spwtmpl.so paper_2007_10752_b200/libtdes_b200.so; do echo "== $so" >> gpurun_out/x.txt; TDES_LIB_PATH=$so python tools/exp/split_tiles.py --mode 0 128 160 256 296 384 >> gpurun_out/x.txt 2>&1; TDES_LIB_PATH=$so python tools/exp/size_timing.py --modes 0 --lo 17 --hi 18 >> gpurun_out/x.txt 2>&1; done
cat gpurun_out/x.txt
