"""B200-native GBEM single-layer Galerkin assembly + SPD solve (arxiv 2203.11733 path).

Native libraries (built in-tree by `python -m paper_2203_11733_b200.build`):
  lib/libgbem_gpu.so   sm_100a kernels behind the C-ABI of include/gbem_gpu.h
  lib/libgbem_host.so  C++ host (scene input, partition, extraction, reports)
The Python layer (api.py) mirrors the reference API and only calls into them.
"""
from .api import (KernelValue, Model, NumericalError, PanelSet, QuadratureConfig, Rect, Span,  # noqa: F401
                  ValidationError, assemble_single, capacitance_matrix, capacitance_row, cholesky_solve,
                  config_model, parse_model, partition_scene, rect, u_pair_integral, u_pair_integrals)

__version__ = "1.0.0"
