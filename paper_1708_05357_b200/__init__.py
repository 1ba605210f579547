"""B200-native DuHL hot path (arXiv 1708.05357): Python binding of libduhl.so.

Argument marshalling only -- every step of the path runs in the library's
sm_100a kernels behind the C ABI declared in ``include/duhl.h``.  The names
mirror the ABI: ``create`` (duhl_create), ``Problem.gaps`` (duhl_gaps),
``Problem.select`` (duhl_select), ``Problem.scd_epoch`` (duhl_scd_epoch),
``Problem.duality_gap`` (duhl_duality_gap), ``Problem.solve`` (duhl_solve);
``create_csc`` (duhl_create_csc) for sparse matrices.

There is no CPU fallback: importing works anywhere (the symbols load), but any
call that computes raises ``DuhlError`` unless a B200 is present.
"""
from ._abi import (LASSO, SVM_DUAL, RIDGE, ELASTIC_NET, SEL_GAP, SEL_SEQUENTIAL, SEL_UNIFORM, SEL_IMPORTANCE, DuhlError, Problem,
                   RoundRecord, Group, create, create_csc, comm_unique_id, lib, lib_path, exported_symbols)

__all__ = ["LASSO", "SVM_DUAL", "RIDGE", "ELASTIC_NET", "SEL_GAP", "SEL_SEQUENTIAL", "SEL_UNIFORM", "SEL_IMPORTANCE", "DuhlError", "Problem",
           "RoundRecord", "Group", "create", "create_csc", "comm_unique_id", "lib", "lib_path", "exported_symbols"]
