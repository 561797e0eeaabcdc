"""Small launches of every kernel, run under compute-sanitizer by tests/test_sanitizer.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402

n = 2 * 1024 + 77                               # two full warp tiles + a ragged tail
s = tdes.key_schedule(*synthetic.KEYS_3KEY)
x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
tdes.fill_splitmix64(x)
y = torch.empty_like(x)
for mode in (1, 2, 3):                            # throughput (host-folded, device-expanded keys) and split kernels
    tdes.ecb_crypt_mode(x, s, mode, out=y)
    tdes.ecb_crypt_mode(y, s, mode, decrypt=True, out=y)   # in place
tdes.ecb_encrypt(x[8:8 + 8 * 1000], s, out=y[8:8 + 8 * 1000])   # 8-byte-aligned path
m = 17 * 1024 + 5                                 # > 16 tiles: the non-specialised split kernel
xm = torch.empty(8 * m, dtype=torch.uint8, device="cuda")
tdes.fill_splitmix64(xm)
tdes.ecb_crypt_mode(xm, s, 2, out=torch.empty_like(xm))
ds = tdes.des_key_schedule(synthetic.KEYS_1KEY[0])
tdes.des_ecb_encrypt(x, ds, out=y)
tdes.PaperBaseline(*synthetic.KEYS_3KEY).run(x[:8 * 64], out=y[:8 * 64])
torch.cuda.synchronize()
print("SANITIZE_TARGET_OK")
