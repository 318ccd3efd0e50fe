"""Generate the seeded inclusion-centre fixtures with the REFERENCE's own sampler.

Test infrastructure (runs only in the build container, where /root/reference
exists).  Calls ``periscat.geometry.place_random_particles``
(/root/reference/pkg/src/periscat/geometry.py:263-314) exactly as SURVEY.md
F5 prescribes and writes ``tests/golden/centers_cfg{N}.npy``.  The GPU box
never runs this; it only reads the committed .npy files.

    PYTHONPATH=/root/reference/pkg/src python oracle/make_geometry.py 1 2 3 5
"""
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from periscat.geometry import (InterfaceSpec, ParticleShape, ProblemConfig,  # noqa: E402
                               place_random_particles)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

# cfg: (M, radius, seed, standoff)   -- BASELINE.json configs, SURVEY F5
GEOM = {
    1: (10, 0.04, 0, 0.02),
    2: (100, 0.04, 1, 0.0),      # standoff 0: 0.02/0.01/0.005 all fail (F5)
    3: (1000, 0.012, 2, 0.02),
    5: (10000, 0.004, 3, 0.002),
}


def make(cfg: int) -> dict:
    m, r, seed, standoff = GEOM[cfg]
    conf = ProblemConfig(period=1.0, k1=10.0, k2=12.0, k3=10.0, kp=15.0,
                         incident_angle=-0.7 * math.pi,
                         interface_top=InterfaceSpec(0.5),
                         interface_bottom=InterfaceSpec(-0.5),
                         seed=seed, particle_shape=ParticleShape(r, 0.0, 1))
    t0 = time.perf_counter()
    ps = place_random_particles(conf, m, standoff)
    dt = time.perf_counter() - t0
    np.save(os.path.join(OUT, f"centers_cfg{cfg}.npy"), ps.centers)
    meta = dict(cfg=cfg, M=m, radius=r, seed=seed, standoff=standoff,
                min_gap=float(ps.min_gap()), seconds=dt,
                numpy=np.__version__, sampler="periscat.geometry.place_random_particles")
    with open(os.path.join(OUT, f"centers_cfg{cfg}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    return meta


if __name__ == "__main__":
    for c in (int(a) for a in sys.argv[1:]):
        print(make(c), flush=True)
