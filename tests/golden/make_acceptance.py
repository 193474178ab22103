"""The reference's own acceptance workload as a golden (TEST INFRASTRUCTURE).

``pkg/tests/test_acceptance.py:60-65,95-121`` (criteria 6b, 7, 8): the P2
tunneling system on [-120, 120] with 4000 elements (7,999 DOF, pentadiagonal),
step barrier 15 / 0.005, packet r = -3, p = 5, sigma = 4, dt = 2e-4, the
flagship K = 16 pole set, 1000 steps.  Run IN THE BUILD CONTAINER (imports the
unmodified reference from /root/reference/pkg/src):

    python tests/golden/make_acceptance.py

Writes tests/golden/acceptance_p2.npz: the system, u0, sr, dt, the reference
states after steps 1, 10, 100 and 1000 of ``rexi_run`` (workers = 1) and its
timings here (prepare and the 1000 steps).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from rexiprop import JoukowskiMap, faber_cf  # noqa: E402
from rexiprop.integrate import rexi_prepare, rexi_run  # noqa: E402
from rexiprop.spatial import (PhysicalConstants, PotentialSpec, WavePacketParams,  # noqa: E402
                              assemble_system, build_mesh, project_initial, spectral_radius_estimate)

DT = 2e-4
CHECK = (1, 10, 100, 1000)


def main():
    consts = PhysicalConstants()
    mesh = build_mesh(-120.0, 120.0, 4000)
    sysm = assemble_system(mesh, PotentialSpec.step_barrier(15.0, 0.005), consts)
    u0 = project_initial(mesh, WavePacketParams(r_bar=-3.0, p_bar=5.0, sigma=4.0), consts, sysm.B)
    flag = faber_cf(JoukowskiMap(10.0))
    sr = float(spectral_radius_estimate(sysm))
    t0 = time.perf_counter()
    stp = rexi_prepare(sysm, flag, DT, workers=1, sr_value=sr)
    t1 = time.perf_counter()
    states = {}
    u = u0
    done = 0
    t_run = 0.0
    for k in CHECK:
        ta = time.perf_counter()
        u = rexi_run(stp, u, k - done)
        t_run += time.perf_counter() - ta
        done = k
        states[k] = u.copy()
    A, B = sysm.A.tocsr(), sysm.B.tocsr()
    out = os.path.join(HERE, "acceptance_p2.npz")
    np.savez_compressed(
        out, A_indptr=A.indptr, A_indices=A.indices, A_data=A.data, A_shape=np.array(A.shape),
        B_indptr=B.indptr, B_indices=B.indices, B_data=B.data, B_shape=np.array(B.shape),
        u0=u0, sr=sr, tau=DT, R1=flag.domain_radius, shifts=flag.shifts, weights=flag.weights,
        check_steps=np.array(CHECK), states=np.stack([states[k] for k in CHECK]),
        bandwidth=stp.factorizations[0].bandwidth, ref_prepare_s=t1 - t0, ref_run_s=t_run,
        admissible=stp.admissible)
    print(f"n {sysm.n_dof} bandwidth {stp.factorizations[0].bandwidth} sr {sr:.4e} admissible "
          f"{stp.admissible}; reference prepare {t1 - t0:.2f} s, 1000 steps {t_run:.2f} s")


if __name__ == "__main__":
    main()
