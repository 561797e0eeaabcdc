"""How a throughput-kernel launch ends: per-warp exit times and tile counts (experiment).

Builds a copy of the library whose tdes_ecb_kernel records, per warp (lane 0), the
%globaltimer at entry, after the prologue, when its last tile ends (exit), the number
of tiles it ran and its SM id; then (on the GPU) reports for each size how much of
the launch the warps spend idle after their last tile (the drain), per SM and overall:

  python tools/exp/trace_drain.py build --out tools/exp/vdrain.so
  TDES_LIB_PATH=tools/exp/vdrain.so python tools/exp/trace_drain.py run [--mode 1] [--sizes 20,22,24,27]
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

GLOBALS = r'''
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
'''


def patch(t: str) -> str:
    t = t.replace("namespace {\n", "namespace {\n" + GLOBALS, 1)
    entry = "  using KT = KeyTable<NSTAGES, DEVKEYS>;\n"
    assert entry in t
    t = t.replace(entry, entry + "  const unsigned long long t_entry = gtimer();\n  unsigned n_done = 0;\n", 1)
    sync = "  expand_keys<NSTAGES, DEVKEYS>(rr, kbits, ksm);\n  __syncthreads();\n"
    assert sync in t
    t = t.replace(sync, sync + "  const unsigned long long t_sync = gtimer();\n", 1)
    loop = "    if (staged) phase ^= 1u;\n"
    assert loop in t
    t = t.replace(loop, loop + "    ++n_done;\n", 1)
    tail = '''    } else {
      tile = claim();
    }
  }
}
'''
    assert tail in t
    t = t.replace(tail, '''    } else {
      tile = claim();
    }
  }
  if (g_trace && lane == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long* p = g_trace + 4ull * (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5));
    p[0] = t_entry; p[1] = t_sync; p[2] = gtimer(); p[3] = ((unsigned long long)smid << 32) | n_done;
  }
}
''', 1)
    return t + '''
extern "C" int tdes_set_trace(void* p) {
  return cudaMemcpyToSymbol(g_trace, &p, sizeof p) == cudaSuccess ? 0 : TDES_ERR_CUDA;
}
'''


def cmd_build(a):
    import __graft_entry__ as ge
    tmp = tempfile.mkdtemp(prefix="tdes_drain_")
    pkg = os.path.join(tmp, "pkg")
    shutil.copytree(ge.CSRC, os.path.join(pkg, "csrc"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    src = os.path.join(pkg, "csrc")
    k = os.path.join(src, "tdes_kernel.cu")
    src_text = open(k).read()
    open(k, "w").write(patch(src_text))
    cmd = [ge._nvcc(), *ge.NVCC_FLAGS, *a.define, "-o", os.path.abspath(a.out), *[os.path.join(src, s) for s in ge.SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr[-3000:])
    print("built", a.out)


def cmd_run(a):
    import ctypes
    import numpy as np
    import torch
    import paper_2007_10752_b200 as tdes
    import synthetic
    lib = tdes._lib
    lib.tdes_set_trace.argtypes = [ctypes.c_void_p]
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    print("log2n tiles | event_us span_us | prologue_end med | warp exit: first/med/last us | "
          "SM drain (last - first warp exit) med/max us | idle warp-time after own exit % | tiles/warp min/max")
    for e in a.sizes:
        n = 1 << e
        x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
        tdes.fill_splitmix64(x)
        y = torch.empty_like(x)
        tr = torch.zeros(4 * sms * 32, dtype=torch.int64, device="cuda")
        for _ in range(3):
            tdes.ecb_crypt_mode(x, s, a.mode, out=y)
        lib.tdes_set_trace(tr.data_ptr())
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(600_000)
        ev0.record()
        tdes.ecb_crypt_mode(x, s, a.mode, out=y)
        ev1.record()
        ev1.synchronize()
        lib.tdes_set_trace(0)
        t = tr.view(-1, 4).cpu().numpy().astype(np.int64)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        ex = (t[:, 2] - t0) / 1e3
        sm = t[:, 3] >> 32
        nd = t[:, 3] & 0xFFFFFFFF
        span = ex.max()
        drains = []
        for m in np.unique(sm):
            e_sm = ex[sm == m]
            drains.append(e_sm.max() - e_sm.min())
        drains = np.array(drains)
        idle = (span - ex).sum() / (span * len(ex)) * 100
        print(f"{e:5d} {n // 1024:6d} | {ev0.elapsed_time(ev1) * 1e3:8.1f} {span:8.1f} | "
              f"{np.median((t[:, 1] - t0) / 1e3):6.2f} | {ex.min():7.1f}/{np.median(ex):7.1f}/{span:7.1f} | "
              f"{np.median(drains):6.1f}/{drains.max():6.1f} | {idle:5.1f} | {nd.min()}/{nd.max()}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("build")
    b.add_argument("--out", required=True)
    b.add_argument("-D", dest="define", action="append", default=[], type=lambda v: "-D" + v)
    r = sub.add_parser("run")
    r.add_argument("--mode", type=int, default=1)
    r.add_argument("--sizes", type=lambda v: [int(x) for x in v.split(",")], default=[19, 20, 21, 22, 23, 24, 27])
    a = ap.parse_args()
    cmd_build(a) if a.cmd == "build" else cmd_run(a)


if __name__ == "__main__":
    main()
