# stagger the warps of each SMSP at start (experiment)
set -x
python tools/exp/ab_sizes.py tools/exp/v_prod.so tools/exp/v_stag500.so tools/exp/v_stag2000.so tools/exp/v_stag5000.so tools/exp/v_prod.so tools/exp/v_stag2000.so > gpurun_out/p_stagger.txt 2>&1
cat gpurun_out/p_stagger.txt
