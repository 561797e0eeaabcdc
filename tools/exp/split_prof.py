import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, paper_2007_10752_b200 as tdes, synthetic
s = tdes.key_schedule(*synthetic.KEYS_3KEY)
x = torch.empty(8 << 17, dtype=torch.uint8, device="cuda"); tdes.fill_splitmix64(x); y = torch.empty_like(x)
for _ in range(3): tdes.ecb_crypt_mode(x, s, 2, out=y)
torch.cuda.synchronize()
