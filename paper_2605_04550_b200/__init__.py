"""B200-native σ_min(zI - A) grid evaluator: drop-in for the hot path of arxiv/paper_2605_04550
(`pseudospec`): smin_many / full_pseudospectrum / restricted_field / hybrid_pseudospectrum.

Submodules:
  core      drop-in for pseudospec.core (σ evaluation through libpsb200.so, grid/field types)
  pipeline  drop-in for the guided path of pseudospec.pipeline (K2 predictor + restricted σ)
  configs   BASELINE.json workloads C1..C5 (seeded bands and grids)
  shim      install(): reroute an imported `pseudospec` package onto this implementation
"""

from .core import (BandMatrix, CalibrationError, ComplexGrid, GenerationError, ModelFormatError,
                   NumericalError, ParameterError, SigmaField, dilate, eigenvalues,
                   full_pseudospectrum, make_grid, restricted_field, sensitive_zone, smin_at,
                   smin_many)

__version__ = "0.1.0"
