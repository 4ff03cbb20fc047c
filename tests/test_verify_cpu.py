"""The output checkers of verify.py (used by bench.py and the -m gpu parity
tests) against the CPU oracle on small cases: they must accept the oracle's
results and reject perturbed ones."""

import numpy as np

import verify
from oracle import bodies, inputs, programs


def test_gemm_checker_accepts_oracle_and_rejects_perturbation():
    n, b = 512, 128
    objs = programs.gemm_operands(n, b)
    programs.run_on_oracle(programs.gemm_program(n // b), objs, workers=2).stop()
    nt = n // b
    A = {(i, k): objs[("A", i, k)] for i in range(nt) for k in range(nt)}
    B = {(i, k): objs[("B", i, k)] for i in range(nt) for k in range(nt)}
    C = {(i, k): objs[("C", i, k)] for i in range(nt) for k in range(nt)}
    samples = verify.sample_tiles(nt, 5)
    rel, comp = verify.gemm_tile_errors(C, A, B, samples)
    assert rel <= verify.GEMM_REL_TOL and comp <= verify.GEMM_COMPONENTWISE_TOL
    C[samples[0]][3, 4] *= 1 + 1e-8
    rel, _ = verify.gemm_tile_errors(C, A, B, samples)
    assert rel > verify.GEMM_REL_TOL


def test_cholesky_residual_accepts_oracle_and_rejects_perturbation():
    n, b = 512, 128
    objs = programs.cholesky_operands(n, b)
    A = {(k[1], k[2]): v.copy() for k, v in objs.items()}
    programs.run_on_oracle(programs.cholesky_program(n // b), objs, workers=2).stop()
    L = {(k[1], k[2]): v for k, v in objs.items()}
    assert verify.cholesky_residual(A, L, n, b) <= verify.CHOL_RESIDUAL_TOL
    L[(2, 1)][5, 6] += 1e-6
    assert verify.cholesky_residual(A, L, n, b) > verify.CHOL_RESIDUAL_TOL


def test_particle_checker_accepts_oracle_and_rejects_perturbation():
    ng, per = 4, 200
    objs = programs.particle_operands(ng, per)
    programs.run_on_oracle(programs.particles_program(ng), objs, workers=2).stop()
    P = [objs[("P", g)] for g in range(ng)]
    F = [objs[("F", g)] for g in range(ng)]
    samples = verify.sample_particles(ng, per, 20)
    pot, force = verify.particle_errors(P, F, samples, eps2=bodies.EPS2, chunk=300)
    assert pot <= verify.POT_REL_TOL and force <= verify.FORCE_NORM_TOL, (pot, force)
    g, a = samples[1]
    F[g][3, a] *= 1 + 1e-8
    F[g][0, a] += 1e-6 * abs(F[g][0, a]) + 1e-6
    pot, force = verify.particle_errors(P, F, samples, eps2=bodies.EPS2)
    assert pot > verify.POT_REL_TOL and force > verify.FORCE_NORM_TOL


def test_spd_input_symmetric_product():
    n, b = 256, 64
    objs = programs.cholesky_operands(n, b)
    A = {(k[1], k[2]): v for k, v in objs.items()}
    dense = programs.assemble_lower(objs, n, b)
    dense = dense + np.tril(dense, -1).T
    X = np.random.default_rng(0).standard_normal((n, 3))
    assert np.allclose(verify._sym_matmul(A, X, b), dense @ X, rtol=1e-13, atol=1e-9)
    assert np.isclose(verify._sym_fro2(A), (dense ** 2).sum())
    assert inputs.spd_tile(3, 0, 0, 4, 4, n).shape == (4, 4)
