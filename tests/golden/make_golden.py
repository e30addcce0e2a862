"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run where /root/reference exists (this container); the fixtures are
committed and the GPU box never needs the reference itself:

    make -C oracle ref && python tests/golden/make_golden.py

Inputs are the reference's keyed generators (seed 1); outputs come from the
FMA-free build of the reference (liblatbench_ref_exact.so, identical
sources) so that the plain-C restatement must reproduce them bit for bit.
Each case stores sha256 digests of the input fields (pinning the RNG and
group algebra) and the full output arrays of Dphi / Mhat / H on a tiny
lattice, plus reference CG iteration counts.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

CASES = [  # name, lattice (T,X,Y,Z), N, rep, mass
    ("su3f", [4, 2, 2, 4], 3, O.FUNDAMENTAL, 0.1),
    ("su2f", [4, 2, 2, 4], 2, O.FUNDAMENTAL, 0.05),
    ("su2a", [4, 2, 2, 4], 2, O.ADJOINT, 0.05),
    ("su4as", [4, 2, 2, 4], 4, O.ANTISYMMETRIC, 0.1),
    ("su3s", [2, 2, 2, 2], 3, O.SYMMETRIC, 0.1),
]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    one = [1, 1, 1, 1]
    with O.exact_reference():
        for name, L, n, rep, m in CASES:
            dr = O.rep_dim(rep, n)
            g = O.ref_gauge_random(L, n, rep, 1)
            s = O.ref_spinor_random(L, dr, 1, 0)
            out = dict(lattice=np.array(L), n=n, rep=rep, mass=m,
                       gauge_sha=sha(g), spinor_sha=sha(s),
                       gauge_first=g.reshape(-1)[:8].copy(), spinor_first=s.reshape(-1)[:8].copy(),
                       dphi_periodic=O.ref_apply_dirac(L, one, n, rep, 0, m, g, s),
                       dphi_antiperiodic=O.ref_apply_dirac(L, one, n, rep, 1, m, g, s),
                       mhat_antiperiodic=O.ref_mhat(L, one, n, rep, 1, m, g, s),
                       h_antiperiodic=O.ref_apply_h(L, one, n, rep, 1, m, g, s))
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
            print(name, "written")
        # BASELINE config 1 exactly: SU(3)F 8^4, m0 = 0.1, antiperiodic t, tol 1e-10
        L = [8, 8, 8, 8]
        g = O.ref_gauge_random(L, 3, O.FUNDAMENTAL, 1)
        s = O.ref_spinor_random(L, 3, 1, 0)
        cg = O.ref_cg_h(L, one, 3, O.FUNDAMENTAL, 1, 0.1, g, s, 1e-10)
        eo = O.ref_cg_eo(L, one, 3, O.FUNDAMENTAL, 1, 0.1, g, s, 1e-10)
        d = O.ref_apply_dirac(L, one, 3, O.FUNDAMENTAL, 1, 0.1, g, s)
        np.savez_compressed(os.path.join(HERE, "cfg1.npz"), lattice=np.array(L), gauge_sha=sha(g),
                            spinor_sha=sha(s), dphi_sha=sha(d), dphi_sqnorm=float(np.vdot(d, d).real),
                            cg_h_iterations=cg["iterations"], cg_h_true=cg["true_rel_residual"],
                            cg_h_history=cg["history"], cg_eo_iterations=eo["iterations"],
                            cg_eo_true=eo["true_rel_residual"], cg_eo_history=eo["history"])
        # near-unit links (config 3 generator, not in the reference: composed on its API)
        nu = O.ref_gauge_near_unit([2, 2, 2, 2], 3, 0.3, 1)
        np.savez_compressed(os.path.join(HERE, "near_unit.npz"), links=nu)
        # group algebra: generators, one Haar element and its representations
        u = O.ref_random_group_element(4, O.ref_key_hash([1, 2]))
        np.savez_compressed(os.path.join(HERE, "group.npz"), gen2=O.ref_generators(2), gen3=O.ref_generators(3),
                            u4=u, u4_adj=O.ref_represent(u, O.ADJOINT), u4_as=O.ref_represent(u, O.ANTISYMMETRIC),
                            u4_s=O.ref_represent(u, O.SYMMETRIC), hop_tables=O.ref_hop_tables(),
                            gammas=O.ref_gamma_matrices())
    print("cfg1 / near_unit / group written")


if __name__ == "__main__":
    main()
