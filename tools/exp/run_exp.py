"""Drive tools/exp/tdes_exp.cu: static vs dynamic tile scheduling, per-warp timelines."""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402

SO = os.path.join(HERE, "libtdes_exp.so")


def build():
    src = os.path.join(HERE, "tdes_exp.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "-Xcompiler", "-fPIC", "-shared", "-cudart", "shared", "-o", SO, src])


def single(mode, launches=3):
    build()
    lib = ctypes.CDLL(SO)
    lib.exp_launch.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 3
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    masks = np.array([[1 if s.mask[0][r][b] else 0 for b in range(48)] for r in range(48)], dtype=np.uint32)
    N = 1 << 27
    x = torch.empty(8 * N, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    sms, occ = tdes.device_geometry()
    grid = sms * occ if mode < 2 else sms
    for _ in range(launches):
        counter.zero_()
        lib.exp_launch(masks.ctypes.data, x.data_ptr(), y.data_ptr(), N // 1024, grid, mode, counter.data_ptr(), 0,
                       torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()


def main():
    if len(sys.argv) > 1:
        return single(int(sys.argv[1]))
    build()
    lib = ctypes.CDLL(SO)
    lib.exp_launch.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 3
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    masks = np.array([[1 if s.mask[0][r][b] else 0 for b in range(48)] for r in range(48)], dtype=np.uint32)
    mp = masks.ctypes.data
    N = 1 << 27
    x = torch.empty(8 * N, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    ref = tdes.ecb_encrypt(x, s)
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    h = torch.cuda.current_stream().cuda_stream
    sms, occ = tdes.device_geometry()
    configs = [(0, sms * occ), (1, sms * occ), (2, sms), (3, sms)]
    names = ["static256", "dyn256", "dyn512", "cta-smem512"]
    ntiles = (1 << 27) // 1024
    res = {c: [] for c in range(len(configs))}
    for rnd in range(4):
        for ci, (mode, grid) in enumerate(configs):
            ts = []
            for rep in range(5):
                counter.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                lib.exp_launch(mp, x.data_ptr(), y.data_ptr(), ntiles, grid, mode, counter.data_ptr(), 0, h)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            ms = sorted(ts)[2]
            res[ci].append((1 << 27) / ms / 1e6)
        print("round", rnd, "  ".join(f"{names[c]}={res[c][-1]:.2f}" for c in res), flush=True)
    assert torch.equal(y, ref)
    # per-warp trace of the smem variant
    trace = torch.zeros(sms * 16 * 4, dtype=torch.int64, device="cuda")
    for mode, grid in ((3, sms), (1, sms * occ)):
        counter.zero_()
        trace.zero_()
        lib.exp_launch(mp, x.data_ptr(), y.data_ptr(), ntiles, grid, mode, counter.data_ptr(), trace.data_ptr(), h)
        torch.cuda.synchronize()
        nw = grid * (16 if mode >= 2 else 8)
        t = trace.view(-1, 4)[:nw].cpu().numpy().astype(np.int64)
        start, end, cyc = t[:, 0], t[:, 1], t[:, 2]
        count = (t[:, 3].astype(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)
        smid = ((t[:, 3].astype(np.uint64) >> np.uint64(32)) & np.uint64(0xFFFF)).astype(np.int64)
        dur = (end - start) / 1e3
        print(f"{names[mode]}: kernel {(end.max() - start.min()) / 1e3:.0f} us; warp dur min {dur.min():.0f} max {dur.max():.0f};"
              f" tiles/warp min {count.min()} max {count.max()}; clk {np.median(cyc / (end - start)):.3f} GHz")
        tiles_sm = np.bincount(smid, weights=count, minlength=sms)
        end_sm = np.array([end[smid == i].max() - start.min() for i in range(sms)]) / 1e3
        print(f"   per-SM tiles min {tiles_sm.min():.0f} max {tiles_sm.max():.0f}; per-SM end us min {end_sm.min():.0f} max {end_sm.max():.0f}")


if __name__ == "__main__":
    main()
