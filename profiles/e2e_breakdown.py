"""Where the end-to-end step time goes (not part of the product): the
host_sync=True path = pointer table + host pack + H2D, GPU step, D2H + host unpack.

    python profiles/e2e_breakdown.py [level]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main(level=4):
    import torch

    from octomini_host import SedovConfig, build_uniform_tree, init_sedov
    from paper_2107_10987_b200 import EosConfig, HydroMode
    from paper_2107_10987_b200.stepper import B200HydroStepper

    t = build_uniform_tree(level, 8, boundary="reflecting")
    init_sedov(SedovConfig(), t, EosConfig(gamma=1.4))
    st = B200HydroStepper(t, EosConfig(gamma=1.4), HydroMode("new"), host_sync=True)
    b = st.batch
    for _ in range(2):
        st.rk3_step(st.cfl_dt(0.4))
    torch.cuda.synchronize()
    host = st._pinned.numpy().reshape(6, b.L + b.nvirtual, 8, 8, 8)
    R = {}

    def tm(name, fn, n=5):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        R[name] = (time.perf_counter() - t0) / n * 1e3

    tm("leaf_ptrs (python)", lambda: b._leaf_ptrs(b.L))
    tm("host_pack", lambda: b.pack(out=host, lib=st.lib))
    tm("h2d", lambda: st._buf[st._state].copy_(st._pinned, non_blocking=True))
    tm("d2h", lambda: st._pinned.copy_(st._buf[st._state]))
    tm("host_unpack", lambda: b.unpack(host, lib=st.lib))
    tm("upload()", st.upload)
    tm("download()", st.download)

    def step():
        st._cfl_launch(0.4)
        st.launch_step(None)
    tm("device step", step)

    def e2e():
        st.rk3_step(st.cfl_dt(0.4))
    tm("e2e step (cfl_dt + rk3_step)", e2e, 3)
    print(f"bytes per copy: {st._pinned.numel() * 8 / 1e6:.1f} MB, host threads {os.cpu_count()}")
    for k, v in R.items():
        print(f"{k:32s} {v:8.2f} ms")


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:2]])
