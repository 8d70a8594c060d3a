"""Host-side octree, EOS helpers, Sedov / star initial data and the checkpoint
reader of octomini (the reference: pkg/src/octomini/mesh/tree.py:26-289,
mesh/transfer.py:13-64, hydro/eos.py:28-77, problems/sedov.py:12-48,
problems/diagnostics.py:9-30, mesh/checkpoint.py:58-114), restated so tests,
``bench.py`` and ``smoke()`` can build the benchmark inputs where octomini is not
importable -- the GPU box (no /root/reference there).  Attribution: the
behaviour, names and error strings are octomini's.  Plus inputs of our own:
the config-c4 AMR Sedov construction, the config-c5 star
stand-in and the smooth non-flat state.

TEST / BENCH INFRASTRUCTURE: the product package (paper_2107_10987_b200)
never imports this; it consumes any tree with octomini's duck type, and
tests/test_octomini_dropin.py drives it with octomini's own trees.
"""

from .eos import conserved_from_primitive, internal_energy, kinetic_energy, pressure, sound_speed  # noqa: F401
from .mesh import Octree, OctreeNode, SubGrid, build_uniform_tree, refine_by_criterion  # noqa: F401
from .problems import (FixedGravity, SedovConfig, amr_sedov_tree, conservation_totals, init_sedov,  # noqa: F401
                       smooth_state, synthetic_star)
