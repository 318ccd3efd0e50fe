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


__all__ = ["SchurOperator", "Solution", "apply_schur_operator", "gmres", "solve_full"]
