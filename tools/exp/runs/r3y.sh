# ptxas --register-usage-level 0/3 (116 regs) and 7/10 (126 regs) vs default 5 (115)
set -x
python tools/exp/ab_variants.py tools/exp/v_rul5.so tools/exp/v_rul0.so tools/exp/v_rul7.so --rounds 3 > gpurun_out/y_rul.txt 2>&1
python tools/exp/ab_sizes.py tools/exp/v_rul5.so tools/exp/v_rul0.so tools/exp/v_rul7.so >> gpurun_out/y_rul.txt 2>&1
python tools/exp/ab_small.py tools/exp/v_rul5.so tools/exp/v_rul0.so tools/exp/v_rul7.so >> gpurun_out/y_rul.txt 2>&1
cat gpurun_out/y_rul.txt
