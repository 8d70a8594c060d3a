"""Wall time of the two public calls of an end-to-end step (not part of the
product): cfl_dt (upload + CFL reduction + dt readback) and rk3_step (three
stages + download), per host-transfer mode.

    python profiles/e2e_timeline.py [level] [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

MODES = [("threads", "0", "1"), ("hybrid", "0.1", "1"), ("threads", "0", "1"), ("hybrid", "0.1", "1"),
         ("hybrid", "0.2", "1")]


def main(level=5, steps=8):
    import numpy as np
    import torch

    from octomini_host import SedovConfig, build_uniform_tree, init_sedov
    from paper_2107_10987_b200 import EosConfig, HydroMode
    from paper_2107_10987_b200.stepper import B200HydroStepper

    for x, f, sc in MODES:
        os.environ.update(OMB_HOST_XFER=x, OMB_GATHER_FRAC=f, OMB_SCATTER_TAIL=sc)
        t = build_uniform_tree(level, 8, boundary="reflecting")
        init_sedov(SedovConfig(), t, EosConfig(gamma=1.4))
        st = B200HydroStepper(t, EosConfig(gamma=1.4), HydroMode("new"), host_sync=True)
        st.rk3_step(st.cfl_dt(0.4))
        a, b = [], []
        for _ in range(steps):
            t0 = time.perf_counter()
            dt = st.cfl_dt(0.4)
            t1 = time.perf_counter()
            st.rk3_step(dt)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            a.append(t1 - t0)
            b.append(t2 - t1)
        c = []
        for _ in range(steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st.upload()
            torch.cuda.synchronize()
            c.append(time.perf_counter() - t0)
        print(f"{x:8s} f={f:4s} scatter={sc}: cfl_dt {np.median(a) * 1e3:7.2f} ms  rk3_step {np.median(b) * 1e3:7.2f} ms"
              f"  (min {min(a) * 1e3:.2f} / {min(b) * 1e3:.2f})  upload() alone {np.median(c) * 1e3:7.2f} ms",
              flush=True)
        del st, t
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:3]])
