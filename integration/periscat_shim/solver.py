"""Drop-in ``periscat.solver`` on top of the reference's
own ``empty_grating`` and ``geometry`` modules.

``solve_full(config)`` follows SPEC.md:559-567: it builds the empty system
with the reference (eg:139-261), places the particles with the reference
sampler (geo:263-314), and runs the coupled solve on the B200.
"""
from __future__ import annotations


from paper_1412_7466_b200.solver import SchurOperator, Solution, apply_schur_operator, gmres  # noqa: F401
from paper_1412_7466_b200.solver import solve_full as _solve_full


def solve_full(config, system=None, particles=None, standoff=None):
    from periscat.empty_grating import assemble_empty_system, factorize
    from periscat.geometry import place_random_particles
    if system is None:
        system = assemble_empty_system(config)
    if system.svd is None:
        factorize(system)
    if particles is None:
        particles = place_random_particles(config, config.particle_count,
                                           config.particle_standoff if standoff is None else standoff)
    shape = particles.shape
    if shape.bump_amplitude != 0.0:
        raise NotImplementedError("general-shape scattering matrices (Mueller BIE) are not built "
                                  "here; pass smat= to paper_1412_7466_b200.solver.solve_full")
    return _solve_full(system, particles.centers, config.multipole_order,
                       radius=shape.base_radius, tol=config.gmres_tol, maxit=config.gmres_maxit)


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


def solve_full_batch(configs, particles, threads: int | None = None):
    """Several incidence angles sharing k2, the period and the particles,
    solved as ONE batch of right-hand sides (BASELINE cfg5: 16 angles): the
    per-angle setup in parallel host threads, then the batched GPU solve
    (multi-RHS M2L on the FP64 tensor cores, batched device GMRES)."""
    systems = assemble_systems(configs, threads)
    shape = particles.shape
    if shape.bump_amplitude != 0.0:
        raise NotImplementedError("general-shape scattering matrices (Mueller BIE) are not built "
                                  "here; pass smat= to paper_1412_7466_b200.solver.solve_full")
    c0 = configs[0]
    return _solve_full(systems, particles.centers, c0.multipole_order, radius=shape.base_radius,
                       tol=c0.gmres_tol, maxit=c0.gmres_maxit)


__all__ = ["SchurOperator", "Solution", "apply_schur_operator", "assemble_systems", "gmres",
           "solve_full", "solve_full_batch"]
