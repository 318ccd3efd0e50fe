"""Drop-in ``periscat.multiscat`` for the reference package.

Copy this file to /path/to/periscat/src/periscat/multiscat.py (the module the
reference's pyproject describes but does not ship) with
paper_1412_7466_b200 importable; the SPEC signatures run on the B200.
"""
from paper_1412_7466_b200.multiscat import apply_T, m2l_translate  # noqa: F401

__all__ = ["apply_T", "m2l_translate"]
