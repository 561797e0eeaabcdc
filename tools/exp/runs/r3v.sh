# split (teams of 4, S-box-specialised) vs throughput kernel at 256..768 tiles: where is the crossover now?
set -x
TDES_LIB_PATH=tools/exp/v_specbig.so python tools/exp/split_tiles.py --mode 2 256 296 320 352 384 448 512 640 768 > gpurun_out/v_cross.txt 2>&1
python tools/exp/split_tiles.py --mode 1 256 296 320 352 384 448 512 640 768 >> gpurun_out/v_cross.txt 2>&1
cat gpurun_out/v_cross.txt
