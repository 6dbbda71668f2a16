"""Generate the first-order comparison numbers for acceptance gate 7.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_gate7.py

Gate 7 of the reference's acceptance suite (tests/test_acceptance.py:342-379)
trains poisson2d (2-32-32-1, 200 iterations) and allen_cahn (3-32x3-1, 300
iterations) with reject_if_worse for seeds 0..9 and compares allen_cahn's D-NGD
loss with the reference's own Adam baseline (`baseline_run(..., "adam", ...)`,
optimizer.py:397).  The Adam runs are a first-order baseline outside this
repository's scope, so their final losses are recorded here from the unmodified
reference and the GPU test (tests/test_gpu_acceptance.py) checks the D-NGD side
on the device against them.  The reference's own D-NGD final numbers are kept
too, as a cross-check of the device runs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from dngd import make_problem  # noqa: E402
from dngd.model import MlpSpec  # noqa: E402
from dngd.optimizer import OptimizerConfig, baseline_run, dngd_run  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SEEDS = range(10)


def main() -> None:
    allen = make_problem("allen_cahn")
    allen_spec = MlpSpec((3, 32, 32, 32, 1))
    allen_cfg = OptimizerConfig(max_iters=300, reject_if_worse=True)
    adam = np.array([baseline_run(allen, allen_spec, "adam", allen_cfg, s).final_loss for s in SEEDS])
    print("adam", adam, flush=True)
    poisson = make_problem("poisson2d")
    poisson_cfg = OptimizerConfig(max_iters=200, reject_if_worse=True)
    ref_poisson = np.array([dngd_run(poisson, MlpSpec((2, 32, 32, 1)), poisson_cfg, s).final_rel_l2
                            for s in SEEDS])
    print("ref poisson rel_l2", ref_poisson, flush=True)
    ref_allen = np.array([dngd_run(allen, allen_spec, allen_cfg, s).final_loss for s in SEEDS])
    print("ref allen loss", ref_allen, flush=True)
    np.savez(os.path.join(HERE, "gate7.npz"), adam_allen_loss=adam,
             ref_poisson_rel_l2=ref_poisson, ref_allen_loss=ref_allen)


if __name__ == "__main__":
    main()
