"""FP64 peaks of this B200 (GPU box): DMMA (mma.sync.m8n8k4.f64) and DFMA throughput from
registers, full grid, best of 5 launches with CUDA events.  Build the probe in the CPU
container first (`python tools/lab/fp64_peaks.py --build`; the .so travels with the
snapshot), then run it on the box; prints one JSON line."""
import ctypes
import json
import os
import subprocess
import sys

LAB = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(LAB, "libfp64_probe.so")


def build():
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", SO,
                           os.path.join(LAB, "fp64_probe.cu")])


def main():
    if "--build" in sys.argv:
        build()
        return
    import torch
    lib = ctypes.CDLL(SO)
    sink = torch.zeros(256, dtype=torch.float64, device="cuda")
    out = {"probe": "fp64 peaks", "gpu": torch.cuda.get_device_name(0)}
    for mode, name in ((0, "dmma_tflops"), (1, "dfma_tflops")):
        best = 0.0
        for cps in (1, 2, 4, 8):
            ms, fl = ctypes.c_float(0), ctypes.c_double(0)
            rc = lib.lab_fp64_probe(mode, cps, 20000, ctypes.c_void_p(sink.data_ptr()),
                                    ctypes.byref(ms), ctypes.byref(fl))
            assert rc == 0, rc
            tf = fl.value / (ms.value * 1e-3) / 1e12
            out["%s_ctas%d" % (name, cps)] = round(tf, 2)
            best = max(best, tf)
        out[name] = round(best, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
