# teams of 4 vs teams of 8 at 128-384 tiles, same box, interleaved x3
set -x
for i in 1 2 3; do for so in v_w8 v_w4; do echo "== $so" >> gpurun_out/ae.txt; TDES_LIB_PATH=tools/exp/$so.so python tools/exp/split_tiles.py --mode 2 128 160 192 256 320 384 >> gpurun_out/ae.txt 2>&1; done; done
cat gpurun_out/ae.txt
