"""Where a throughput-kernel launch spends its time outside the rounds (experiment).

Builds a copy of the library whose tdes_ecb_kernel records %globaltimer per warp
(lane 0) at kernel entry, after its own share of the key expansion, after the
prologue's final __syncthreads and at exit, then (on the GPU) times single launches
with CUDA events beside the traced span:

  python tools/exp/trace_prologue.py build --out tools/exp/vtrace.so
  TDES_LIB_PATH=tools/exp/vtrace.so python tools/exp/trace_prologue.py run [--mode 1]
"""
import argparse
import ctypes
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

PATCH_GLOBALS = r'''
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
'''


def cmd_build(a):
    import __graft_entry__ as ge
    tmp = tempfile.mkdtemp(prefix="tdes_trace_")
    pkg = os.path.join(tmp, "pkg")
    shutil.copytree(ge.CSRC, os.path.join(pkg, "csrc"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    src = os.path.join(pkg, "csrc")
    k = os.path.join(src, "tdes_kernel.cu")
    t = open(k).read()
    t = t.replace("namespace {\n", "namespace {\n" + PATCH_GLOBALS, 1)
    entry = "  using KT = KeyTable<NSTAGES, DEVKEYS>;\n"
    assert entry in t
    t = t.replace(entry, entry + "  const unsigned long long t_entry = gtimer();\n", 1)
    copy = "  expand_keys<NSTAGES, DEVKEYS>(rr, kbits, ksm);\n  __syncthreads();\n"
    assert copy in t
    t = t.replace(copy, "  expand_keys<NSTAGES, DEVKEYS>(rr, kbits, ksm);\n  const unsigned long long t_copy = gtimer();\n"
                  "  __syncthreads();\n  const unsigned long long t_sync = gtimer();\n", 1)
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
    unsigned long long* p = g_trace + 4ull * (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5));
    p[0] = t_entry; p[1] = t_sync; p[2] = gtimer(); p[3] = t_copy;
  }
}
''', 1)
    t += '''
extern "C" int tdes_set_trace(void* p) {
  return cudaMemcpyToSymbol(g_trace, &p, sizeof p) == cudaSuccess ? 0 : TDES_ERR_CUDA;
}
'''
    open(k, "w").write(t)
    cmd = [ge._nvcc(), *ge.NVCC_FLAGS, "-o", os.path.abspath(a.out), *[os.path.join(src, s) for s in ge.SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr[-3000:])
    print("built", a.out)


def cmd_run(a):
    import numpy as np
    import torch
    import paper_2007_10752_b200 as tdes
    import synthetic
    lib = tdes._lib
    lib.tdes_set_trace.argtypes = [ctypes.c_void_p]
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    print("log2n tiles | event_us(queued) span_us | prologue_us med/max | key copy us med/max | entry spread_us | exit spread_us")
    for e in a.sizes:
        n = 1 << e
        x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
        tdes.fill_splitmix64(x)
        y = torch.empty_like(x)
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        tr = torch.zeros(4 * sms * 16, dtype=torch.int64, device="cuda")
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
        pro = (t[:, 1] - t[:, 0]) / 1e3
        cp = (t[:, 3] - t[:, 0]) / 1e3
        print(f"{e:5d} {n // 1024:6d} | {ev0.elapsed_time(ev1) * 1e3:9.1f} {(t[:, 2].max() - t0) / 1e3:8.1f} | "
              f"{np.median(pro):6.2f}/{pro.max():6.2f} | {np.median(cp):6.2f}/{cp.max():6.2f} | "
              f"{(t[:, 0].max() - t0) / 1e3:8.2f} | "
              f"{(t[:, 2].max() - t[:, 2].min()) / 1e3:8.1f}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("build")
    b.add_argument("--out", required=True)
    r = sub.add_parser("run")
    r.add_argument("--mode", type=int, default=1)
    r.add_argument("--sizes", type=lambda v: [int(x) for x in v.split(",")], default=[14, 17, 19, 20, 21, 22, 27])
    a = ap.parse_args()
    cmd_build(a) if a.cmd == "build" else cmd_run(a)


if __name__ == "__main__":
    main()
