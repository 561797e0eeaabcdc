"""Experiment: per-block cost vs launch size (why is a 1 GiB launch slower than 256 MiB?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402


def med_time(fn, reps=15, warm=3):
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
    return ts[len(ts) // 2], ts[0]


def main():
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    N = 1 << 27
    x = torch.empty(8 * N, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    h = torch.cuda.current_stream().cuda_stream
    for e in (22, 23, 24, 25, 26, 27):
        n = 1 << e
        med, mn = med_time(lambda: tdes.ecb_encrypt_ptr(s, x.data_ptr(), y.data_ptr(), n, h))
        print(f"single 2^{e}: med {med:.3f} ms min {mn:.3f}  -> {n / med / 1e6:.2f} Gblk/s (per-block ns {med * 1e6 / n:.4f})")
    for e in (23, 25):
        n = 1 << e
        parts = N // n

        def split():
            for p in range(parts):
                tdes.ecb_encrypt_ptr(s, x.data_ptr() + 8 * n * p, y.data_ptr() + 8 * n * p, n, h)
        med, mn = med_time(split, reps=7)
        print(f"2^27 as {parts} x 2^{e}: med {med:.3f} ms -> {N / med / 1e6:.2f} Gblk/s")
    # same 2^25 region repeated 4x (is it address-range dependent?)
    n = 1 << 25

    def same():
        for p in range(4):
            tdes.ecb_encrypt_ptr(s, x.data_ptr(), y.data_ptr(), n, h)
    med, mn = med_time(same, reps=7)
    print(f"4 x 2^25 same region: med {med:.3f} ms -> {4 * n / med / 1e6:.2f} Gblk/s")
    # in-place
    med, mn = med_time(lambda: tdes.ecb_encrypt_ptr(s, x.data_ptr(), x.data_ptr(), N, h))
    print(f"2^27 in place: med {med:.3f} ms -> {N / med / 1e6:.2f} Gblk/s")


if __name__ == "__main__":
    main()
