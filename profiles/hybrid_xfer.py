"""Host-transfer split experiment (not part of the product): with the leaves
re-homed in the mapped pinned slab, move a fraction f of them with the GPU's
zero-copy kernels (omb_host_gather / omb_host_scatter, on a side stream) and
the rest with host threads + DMA (omb_host_upload / omb_host_download), at the
same time.  Prints ms per full-state transfer for each f.

    python profiles/hybrid_xfer.py [level]
"""
import os
import sys
import time

os.environ["OMB_HOST_XFER"] = "mapped"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main(level=5):
    import ctypes

    import torch

    from octomini_host import SedovConfig, build_uniform_tree, init_sedov
    from paper_2107_10987_b200 import EosConfig, HydroMode
    from paper_2107_10987_b200.device import ptr, stream_handle
    from paper_2107_10987_b200.stepper import B200HydroStepper

    t = build_uniform_tree(level, 8, boundary="reflecting")
    init_sedov(SedovConfig(), t, EosConfig(gamma=1.4))
    st = B200HydroStepper(t, EosConfig(gamma=1.4), HydroMode("new"), host_sync=True)
    b = st.batch
    lib = st.lib
    m = st._mapped
    assert m is not None
    nc = b.ncompute
    dev = st._buf[st._state]
    pinned = torch.zeros(6 * b.fstride, dtype=torch.float64).pin_memory()
    hptrs = b._leaf_ptrs(nc)
    side = torch.cuda.Stream()
    main_s = torch.cuda.current_stream()
    SS = st.SPAN_STASH

    def up(f):
        k = int(round(nc * (1 - f)))
        if k < nc:
            side.wait_stream(main_s)
            lib.omb_host_gather(ptr(m["ptrs"]) + 8 * k, nc - k, b.fstride, ptr(dev) + 8 * 512 * k,
                                ptr(m["stash"]) + 8 * SS * k, ctypes.c_void_p(side.cuda_stream))
        if k > 0:
            lib.omb_host_upload(hptrs.ctypes.data, k, 8, 14, b.fstride, ptr(pinned), ptr(dev), 8, stream_handle(None))
        main_s.wait_stream(side)

    def down(f):
        k = int(round(nc * (1 - f)))
        if k < nc:
            side.wait_stream(main_s)
            lib.omb_host_scatter(ptr(dev) + 8 * 512 * k, ptr(m["stash"]) + 8 * SS * k, nc - k, b.fstride,
                                 ptr(m["ptrs"]) + 8 * k, ctypes.c_void_p(side.cuda_stream))
        if k > 0:
            lib.omb_host_download(ptr(dev), ptr(pinned), k, 8, 14, b.fstride, hptrs.ctypes.data, 8, stream_handle(None))
        side.synchronize()

    def tm(fn, n=5):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / n * 1e3

    print(f"level {level}: {nc} leaves, {6 * nc * 512 * 8 / 1e6:.1f} MB each way, cpu_count {os.cpu_count()}")
    for f in (0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.7, 1.0):
        print(f"f={f:.1f}  upload {tm(lambda: up(f)):7.2f} ms   download {tm(lambda: down(f)):7.2f} ms", flush=True)


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:2]])
