"""Per-phase cycle breakdown of k_stage (profiling build only, not the product):

    python -c "from paper_2107_10987_b200 import build; build.build(force=True, out='exp/lib_prof.so', defines=('OMB_PHASE_PROF',))"
    OMB_LIB_PATH=exp/lib_prof.so python profiles/phase_prof.py [sedov|smooth] [level] [steps]

Thread 0 of every CTA reads clock64() after each barrier; the cycles between
barrier exits are summed per phase over planes and CTAs."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
NAMES = ["prologue", "P0 convert + P5 of prev plane", "P1A lines 0,3-6 + KT", "P2A combine",
         "P1B lines 9-12 + KT", "P2B combine", "P3 in-plane mono + P6", "P4 in-plane KT", "last P5",
         "epilogue P6"]


def main(kind="sedov", level=4, steps=3):
    import torch

    from octomini_host import SedovConfig, build_uniform_tree, init_sedov
    from paper_2107_10987_b200 import EosConfig, HydroMode
    from octomini_host import smooth_state
    from paper_2107_10987_b200.stepper import B200HydroStepper

    t = build_uniform_tree(level, 8, boundary="reflecting")
    init_sedov(SedovConfig(), t, EosConfig(gamma=1.4))
    if kind == "smooth":
        t = smooth_state(t)
    st = B200HydroStepper(t, EosConfig(gamma=1.4), HydroMode("new"), host_sync=False)
    lib = st.lib
    buf = (ctypes.c_ulonglong * 16)()
    st._cfl_launch(0.4)
    st.launch_step(None)
    torch.cuda.synchronize()
    lib.omb_phase_prof(buf, 1)
    for _ in range(steps):
        st._cfl_launch(0.4)
        st.launch_step(None)
    torch.cuda.synchronize()
    lib.omb_phase_prof(buf, 1)
    tot = sum(buf[i] for i in range(10))
    print(f"{kind} L{level}, {steps} steps: {tot / 1e9:.3f} G CTA-cycles")
    for i, n in enumerate(NAMES):
        print(f"  {n:28s} {100 * buf[i] / tot:5.1f} %")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "sedov", *[int(x) for x in a[1:3]])
