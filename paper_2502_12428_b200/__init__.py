"""B200-native batched quasi-F-split heights of quartic K3 surfaces (drop-in for qfsplit's hot path).

The names below mirror the reference package's flat export list (qfsplit/__init__.py:11-114) for the
path this package replaces; heights come from hand-written sm_100a kernels behind libqfs.so
(include/qfs.h).  There is no CPU fallback: without the library or a GPU the compute entry points
raise EngineUnavailableError.
"""
from .cubic import Cubic, cubic_height_batch
from .forms import Form, form_height_batch
from .literal import literal_heights
from .errors import DomainError, EngineUnavailableError, InternalInvariantError, ParseError, QfsplitError
from .height import (INFINITE, HeightResult, SurfaceProblem, default_bound, height_batch, height_matrix,
                     height_naive, height_of_coeffs, is_prime)
from .mtsmatrix import (MtsMatrix, build_mts, build_mts_batch, matrix_from_bytes, matrix_from_text, matrix_to_bytes,
                        matrix_to_text, target_degree)
from .quartic import Quartic, coeff_vector, parse_poly, poly_to_text
from .stages import DenseForm, DenseVector, delta1, fedder_survives, matvec, power_mod_p, to_dense
from .search import (FixtureRow, FixtureVerdict, FoundSurface, HeightHistogram, SearchConfig, found_surfaces_text,
                     histogram_text, parse_fixtures, run_search, sample_block, sample_surface, spectrum_rows,
                     spectrum_search, verify_fixtures)

__version__ = "0.1.0"


def fixtures_path() -> str:
    """Location of the packaged table of known surfaces (search.py:157-159)."""
    import os
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "fixtures", "k3_tables.txt")


__all__ = [
    "DomainError", "EngineUnavailableError", "InternalInvariantError", "ParseError", "QfsplitError",
    "INFINITE", "HeightResult", "SurfaceProblem", "default_bound", "height_batch", "height_matrix",
    "height_naive", "height_of_coeffs", "is_prime", "Quartic", "coeff_vector", "parse_poly", "poly_to_text",
    "FixtureRow", "FixtureVerdict", "FoundSurface", "HeightHistogram", "SearchConfig", "found_surfaces_text",
    "histogram_text", "parse_fixtures", "run_search", "sample_block", "sample_surface", "spectrum_rows",
    "spectrum_search", "verify_fixtures", "fixtures_path",
    "Cubic", "cubic_height_batch", "Form", "form_height_batch", "literal_heights", "MtsMatrix", "build_mts", "build_mts_batch", "matrix_from_bytes", "matrix_from_text", "matrix_to_bytes",
    "matrix_to_text", "target_degree",
    "DenseForm", "DenseVector", "delta1", "fedder_survives", "matvec", "power_mod_p", "to_dense",
]
