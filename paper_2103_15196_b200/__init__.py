"""B200-native CSPH-TVD shallow water + Exner step (arXiv 2103.15196).

The product path: ``libcsph.so`` (CUDA kernels for sm_100a behind the C-ABI of
``include/csph.h``) and its thin ctypes binding ``csph``.
"""
from .csph import (  # noqa: F401
    CSPH_PATH_FUSED, CSPH_PATH_STAGED, Csph, CsphError, csph_create, csph_create_dist,
    csph_create_multi, csph_default_params, csph_make_nccl_id, csph_nccl_id_bytes,
    csph_strip_rows, params_from,
)
