"""Drop-in ``periscat.solver`` on top of the reference's
own ``empty_grating`` and ``geometry`` modules.

``solve_full(config)`` follows SPEC.md:559-567: it places the particles with
the reference sampler (geo:263-314) and runs everything else on the B200: the
empty-grating assembly and SVD (ps_setup_empty, replacing eg:139-261), the
particle scattering matrix (the analytic disk, or the Mueller BIE for star
shapes via ps_scattering_matrix), and the coupled solve.  ``setup="host"``
keeps the reference's own host assembly + numpy SVD instead.
"""
from __future__ import annotations


from paper_1412_7466_b200.solver import SchurOperator, Solution, apply_schur_operator, gmres  # noqa: F401
from paper_1412_7466_b200.solver import solve_full as _solve_full


def _particle_smatrix(config, particles):
    """(smat, radius, rot) for the solver: the disk's analytic diagonal, or
    the device Mueller-BIE matrix of a star shape with the
    particles' rotations."""
    from paper_1412_7466_b200 import scatmat
    shape = particles.shape
    if shape.bump_amplitude == 0.0:
        return None, shape.base_radius, None
    sm = scatmat.scattering_matrix(shape, config.k2, config.kp, config.multipole_order,
                                   N=config.particle_nodes, alpert_order=config.alpert_order)
    return sm, None, particles.rotations


def solve_full(config, system=None, particles=None, standoff=None, setup: str = "device"):
    from periscat.geometry import place_random_particles
    if particles is None:
        particles = place_random_particles(config, config.particle_count,
                                           config.particle_standoff if standoff is None else standoff)
    if system is None and setup == "host":
        system = _assemble_factorize(config)
    if system is not None and system.svd is None:
        from periscat.empty_grating import factorize
        factorize(system)
    smat, radius, rot = _particle_smatrix(config, particles)
    return _solve_full(config if system is None else system, particles.centers,
                       config.multipole_order, radius=radius, smat=smat, rot=rot,
                       tol=config.gmres_tol, maxit=config.gmres_maxit)


def _assemble_factorize(config):
    from periscat.empty_grating import assemble_empty_system, factorize
    system = assemble_empty_system(config)
    factorize(system)
    return system


def assemble_systems(configs, threads: int | None = None):
    """Empty-grating systems + SVDs for several incidence angles (SURVEY 8f
    row 1: setup off the critical path).  The reference assembly (eg:139-261)
    is host NumPy/SciPy, ~2.7 s + 0.36 s SVD per angle.  The angles are
    independent and the systems hold closures (no pickling to processes), so
    they run in threads: SciPy's special-function ufuncs and LAPACK release
    the GIL (3.6x on 8 threads here)."""
    import concurrent.futures as cf
    import os
    configs = list(configs)
    n = min(len(configs), threads or os.cpu_count() or 1)
    if n <= 1:
        return [_assemble_factorize(c) for c in configs]
    with cf.ThreadPoolExecutor(n) as ex:
        return list(ex.map(_assemble_factorize, configs))


def solve_full_batch(configs, particles, threads: int | None = None, setup: str = "device"):
    """Several incidence angles sharing k2, the period and the particles,
    solved as ONE batch of right-hand sides (BASELINE cfg5: 16 angles): the
    per-angle empty-grating setup (one device assembly launch + concurrent
    cuSOLVER SVDs, or ``setup="host"``: the reference assembly in parallel host
    threads), then the batched GPU solve (multi-RHS M2L on the FP64 tensor
    cores, batched device GMRES)."""
    configs = list(configs)
    systems = assemble_systems(configs, threads) if setup == "host" else configs
    c0 = configs[0]
    smat, radius, rot = _particle_smatrix(c0, particles)
    return _solve_full(systems, particles.centers, c0.multipole_order, radius=radius, smat=smat,
                       rot=rot, tol=c0.gmres_tol, maxit=c0.gmres_maxit)


__all__ = ["SchurOperator", "Solution", "apply_schur_operator", "assemble_systems", "gmres",
           "solve_full", "solve_full_batch"]
