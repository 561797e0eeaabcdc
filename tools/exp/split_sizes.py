"""Forced split-kernel launches at a few sizes (for ncu duration captures)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402

s = tdes.key_schedule(*synthetic.KEYS_3KEY)
x = torch.empty(8 << 18, dtype=torch.uint8, device="cuda")
tdes.fill_splitmix64(x)
y = torch.empty_like(x)
for e in (10, 14, 17, 18):
    for _ in range(2):
        tdes.ecb_crypt_mode(x[:8 << e], s, 2, out=y[:8 << e])
torch.cuda.synchronize()
