"""Quick device timing of the 3DES kernel and the LOP3 peak (dev aid, not the bench)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402


def time_it(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    sms, occ = tdes.device_geometry()
    print("SMs", sms, "ctas/SM", occ, "kernel", tdes.kernel_info().sbox_lop3_total)
    sink = torch.empty(sms * 8 * 256, dtype=torch.int32, device="cuda")
    for grid_mult, iters in ((8, 4096), (8, 16384)):
        grid = sms * grid_mult
        ops = [0]

        def run():
            ops[0] = tdes.lop3_peak_launch(sink, grid, 256, iters)
        ms = time_it(run)
        print(f"lop3 peak grid={grid} iters={iters}: {ops[0] / ms / 1e9:.3f} Tops/s ({ms:.3f} ms)")
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    for e in (17, 20, 23, 25, 27):
        n = 1 << e
        x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
        tdes.fill_splitmix64(x)
        y = torch.empty_like(x)
        ms = time_it(lambda: tdes.ecb_encrypt(x, s, out=y))
        print(f"3DES enc 2^{e} blocks: {ms:.3f} ms  {n * 8 / ms / 1e6:.1f} GB/s  {n / ms / 1e6:.3f} Gblk/s")
        del x, y
    base = tdes.PaperBaseline(*synthetic.KEYS_3KEY)
    for e in (17, 20, 23):
        n = 1 << e
        x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
        tdes.fill_splitmix64(x)
        y = torch.empty_like(x)
        ms = time_it(lambda: base.run(x, out=y), reps=5)
        print(f"paper-design kernel 2^{e} blocks: {ms:.3f} ms  {n * 8 / ms / 1e6:.2f} GB/s")
    ds = tdes.des_key_schedule(synthetic.KEYS_1KEY[0])
    n = 1 << 27
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    ms = time_it(lambda: tdes.des_ecb_encrypt(x, ds, out=y))
    print(f"DES enc 2^27 blocks: {ms:.3f} ms  {n * 8 / ms / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
