"""Minimal driver for ncu captures of the 3DES kernel: the bench workload (1 GiB
encrypt, 3-key), a few launches.  Usage under ncu:

  ncu --set full --clock-control none --import-source on -k regex:tdes_ecb_kernel \
      -s 2 -c 1 -o gpurun_out/prof python tools/profile_kernel.py [--log2n 27] [--op enc|dec|des] [--keys 2key]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=27)
    ap.add_argument("--op", default="enc", choices=["enc", "dec", "des"])
    ap.add_argument("--launches", type=int, default=4)
    ap.add_argument("--mode", type=int, default=None, help="force a 3DES kernel (tdes_ecb_crypt_mode)")
    ap.add_argument("--keys", default="3key", choices=["3key", "2key", "1key"], help="keying (C3: 2key/1key)")
    a = ap.parse_args()
    n = 1 << a.log2n
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    s = tdes.key_schedule(*{"3key": synthetic.KEYS_3KEY, "2key": synthetic.KEYS_2KEY,
                            "1key": synthetic.KEYS_1KEY}[a.keys])
    ds = tdes.des_key_schedule(synthetic.KEYS_1KEY[0])
    for _ in range(a.launches):
        if a.mode is not None and a.op in ("enc", "dec"):
            tdes.ecb_crypt_mode(x, s, a.mode, decrypt=a.op == "dec", out=y)
        elif a.op == "enc":
            tdes.ecb_encrypt(x, s, out=y)
        elif a.op == "dec":
            tdes.ecb_decrypt(x, s, out=y)
        else:
            tdes.des_ecb_encrypt(x, ds, out=y)
    torch.cuda.synchronize()
    print("done", n)


if __name__ == "__main__":
    main()
