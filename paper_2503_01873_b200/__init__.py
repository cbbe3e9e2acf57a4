"""B200-native PASA forward (arXiv 2503.01873): pseudo-average shifting attention
with FP16 tensor-core GEMMs and an FP16 online softmax, drop-in for the
reference's ``pasa::pasa_attention`` operator.

The compute lives in ``libpasa_b200.so`` (CUDA, sm_100a, C-ABI in
``include/pasa_b200.h``); this package is the Python host mirror of the
reference's operator API.
"""
from .api import (BETA_STAR, AttentionProblem, AttnOptions, M0Mode, PasaParams, PolicyId, Prec,
                  PrecisionPolicy, RunDiagnostics, SingularMatrixError, build_shifting_matrix,
                  flash_attention, flash_fp16_fwd, make_problem, pasa_attention, pasa_attention_fwd,
                  policy_for, preprocess_keys, shift_entries, shifting_matrix_inverse)

__all__ = [
    "BETA_STAR", "AttentionProblem", "AttnOptions", "M0Mode", "PasaParams", "PolicyId", "Prec",
    "PrecisionPolicy", "RunDiagnostics", "SingularMatrixError", "build_shifting_matrix", "flash_attention",
    "flash_fp16_fwd", "make_problem", "pasa_attention",
    "pasa_attention_fwd", "policy_for", "preprocess_keys", "shift_entries", "shifting_matrix_inverse",
]
