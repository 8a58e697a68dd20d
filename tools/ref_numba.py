"""Times the UNMODIFIED reference (svdlut in baseline/_ref, numba) on the host
cores — the CPU side of bench.py's reference arm (SURVEY.md §8d protocol).

    python tools/ref_numba.py fused  --threads N --frames F   # config 2, 4K
    python tools/ref_numba.py model  --frames F               # config 1, run_model 720x480

Run each mode in a FRESH process with a FRESH NUMBA_CACHE_DIR (bench.py does):
the serial and parallel numba twins share one on-disk cache entry
(transform.py:303-305), so the parallel twin is compiled and called first.
Prints one JSON line: MP/s over the timed frames (public API), kernel-only
MP/s (the numba twin on preallocated buffers), threads, compile seconds.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["fused", "model"])
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--frames", type=int, default=3)
    a = ap.parse_args()
    if not os.path.isdir(os.path.join(REF, "svdlut")):
        print(json.dumps({"unavailable": "reference not installed in baseline/_ref (tools/install_reference.sh)"}))
        return 0
    sys.path.insert(0, REF)
    sys.path.insert(1, ROOT)
    sys.dont_write_bytecode = True
    import numba
    from svdlut import network, svd, transform
    from svdlut.core_types import GridSet, GridWeights, Image, LutWeights, SvdLut

    from paper_2508_16121_b200 import synth

    if a.mode == "model":  # config 1: the full reference model forward, single image
        rng = np.random.default_rng(0)
        img = Image(720, 480, rng.random((3, 480, 720), dtype=np.float32))
        params = network.random_init(0)
        t0 = time.perf_counter()
        network.run_model(img, params, threads=a.threads)  # JIT + warm-up
        comp = time.perf_counter() - t0
        times = []
        for _ in range(a.frames):
            t0 = time.perf_counter()
            network.run_model(img, params, threads=a.threads)
            times.append(time.perf_counter() - t0)
        print(json.dumps({"mode": "model", "threads": a.threads, "ms_median": 1e3 * float(np.median(times)),
                          "mps": 720 * 480 / float(np.median(times)) / 1e6, "warmup_s": comp,
                          "numba": numba.__version__}))
        return 0

    case = synth.make_case(0)
    h, w = case.rgb.shape[1:]
    img = Image(w, h, case.rgb)
    factors = SvdLut(case.u, case.s, case.vt)
    lw = LutWeights(case.lw, case.lb)
    grids, gw = GridSet(case.grid_planes), GridWeights(case.gw, case.gb)
    luts = svd.reconstruct_lut(factors)
    threads = min(a.threads, numba.config.NUMBA_NUM_THREADS)
    t0 = time.perf_counter()
    transform.fused_enhance(img, luts, lw, grids, gw, threads=threads)  # compiles the twin in use first
    comp = time.perf_counter() - t0
    api = []
    for _ in range(a.frames):  # public API: reconstruct + fused_enhance (incl. output validation)
        t0 = time.perf_counter()
        transform.fused_enhance(img, svd.reconstruct_lut(factors), lw, grids, gw, threads=threads)
        api.append(time.perf_counter() - t0)
    ix, dx, iy, dy = transform._spatial_brackets(w, h, grids.d_s)
    out = np.empty((3, h, w), np.float32)
    args = (img.data, luts.planes, lw.w, lw.b, grids.planes, gw.w, gw.b, ix, dx, iy, dy, out)
    twin = transform._fused_parallel if threads > 1 else transform._fused_serial
    if threads > 1:
        numba.set_num_threads(threads)
    kern = []
    for _ in range(a.frames):
        t0 = time.perf_counter()
        twin(*args)
        kern.append(time.perf_counter() - t0)
    print(json.dumps({"mode": "fused", "threads": threads, "frames": a.frames,
                      "mps": h * w / float(np.median(api)) / 1e6, "kernel_mps": h * w / float(np.median(kern)) / 1e6,
                      "ms_median": 1e3 * float(np.median(api)), "compile_s": comp, "numba": numba.__version__}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
