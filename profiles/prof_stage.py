"""Profiling driver (not part of the product): a few steps of k_stage on a
level-3 tree (512 leaves = 128 runs, one wave) for ncu, Sedov or smooth state.

    ncu --set full --import-source on -k regex:k_stage -s 6 -c 1 python profiles/prof_stage.py sedov
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main(kind="sedov", level=3, steps=3):
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
    for _ in range(steps):
        st._cfl_launch(0.4)
        st.launch_step(None)
    torch.cuda.synchronize()
    print("ok", kind, level, steps)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["sedov"]), *[int(a) for a in sys.argv[2:4]])
