"""ctypes binding of libpathfield_b200.so (the C ABI in include/pathfield_b200.h).

There is no CPU fallback: if the library is missing, or no CUDA device is
visible, every device entry point raises.  ``symbols()`` lists the exported
names so the CPU test-suite can check that the library loads and exports
every declaration of the header without launching anything.
"""

from __future__ import annotations

import ctypes
import re
import threading
from pathlib import Path

from .errors import NativeError

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libpathfield_b200.so"
HEADER = PKG.parent / "include" / "pathfield_b200.h"

_lock = threading.Lock()
_lib = None

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p

# name -> argtypes (all return int unless listed in _RESTYPES)
_SIGS = {
    "pf_version": [],
    "pf_last_error": [],
    "pf_sm_count": [],
    "pf_target_prep_f64": [c_vp, c_i64, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp],
    "pf_row_negentropy_f64": [c_vp, c_i64, c_i64, c_i64, c_dbl, c_vp, c_vp, c_vp],
    "pf_dense_kl_f64": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_dbl, c_dbl,
                        c_i64, c_i64, c_vp, c_vp, c_vp, c_vp],
    "pf_dense_tv_f64": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_dbl, c_i64, c_i64, c_vp,
                        c_vp, c_vp, c_vp],
    "pf_dense_generic_f64": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_dbl, c_int, c_dbl,
                             c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp],
    "pf_dense_at_f64": [c_vp, c_i64, c_i64, c_i64, c_vp, c_dbl, c_int, c_dbl, c_int, c_i64,
                        c_i64, c_vp, c_i64, c_vp, c_vp],
    "pf_csr_count_f64": [c_vp, c_i64, c_i64, c_i64, c_dbl, c_int, c_vp, c_vp],
    "pf_csr_fill_f64": [c_vp, c_i64, c_i64, c_i64, c_dbl, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                        c_vp, c_vp],
    "pf_csr_target_prep_f64": [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp],
    "pf_csr_kl_f64": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_dbl, c_i64, c_vp,
                      c_i64, c_vp, c_vp, c_vp, c_int, c_vp],
    "pf_csr_tv_f64": [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64,
                      c_vp, c_vp, c_vp],
    "pf_csr_kl_u16_f64": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_dbl, c_i64, c_vp,
                          c_i64, c_vp, c_vp, c_vp, c_int, c_vp],
    "pf_csr_tv_u16_f64": [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64,
                      c_vp, c_vp, c_vp],
    "pf_csr_narrow_u16": [c_vp, c_i64, c_vp, c_vp],
    "pf_csr_unpad": [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "pf_log_clamped_f64": [c_vp, c_i64, c_i64, c_i64, c_dbl, c_vp, c_vp],
    "pf_csr_generic_f64": [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_dbl, c_dbl, c_vp,
                           c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp],
    "pf_batch_prep_f64": [c_vp, c_i64, c_i64, c_i64, c_i64, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp],
    "pf_mask_uniform_f64": [c_vp, c_i64, c_i64, c_i64, c_dbl, c_vp, c_vp, c_vp, c_vp],
    "pf_batched_kl_f64": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_dbl,
                          c_dbl, c_i64, c_vp, c_i64, c_vp, c_vp],
    "pf_batched_kl_fixup_f64": [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_dbl, c_vp,
                                c_i64, c_vp, c_vp],
    "pf_batched_kl_fixup_list_f64": [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_i64, c_dbl,
                                     c_vp, c_i64, c_vp, c_vp, c_i64, c_vp],
    "pf_slice_rows_u8": [c_vp, c_i64, c_i64, c_i64, c_dbl, c_i64, c_vp, c_vp, c_vp],
    "pf_slice_targets_u8": [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp],
    "pf_batched_kl_i8": [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_dbl,
                         c_i64, c_vp, c_i64, c_int, c_int, c_vp],
    "pf_batched_kl_i8_listed": [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp,
                                c_dbl, c_i64, c_vp, c_i64, c_int, c_int, c_vp, c_i64, c_vp],
    "pf_i8_tiled_bytes": [c_i64, c_i64],
    "pf_slice_rows_u8_tiled": [c_vp, c_i64, c_i64, c_i64, c_dbl, c_vp, c_vp, c_vp],
    "pf_slice_targets_u8_tiled": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp],
    "pf_batched_kl_i8_tiled": [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_dbl,
                               c_i64, c_vp, c_i64, c_int, c_vp, c_i64, c_vp],
    "pf_probe_umma_i8": [c_i64, c_int, ctypes.POINTER(ctypes.c_int64), c_vp, c_vp],
    "pf_probe_dfma_f64": [c_i64, ctypes.POINTER(ctypes.c_int64), c_vp, c_vp],
    "pf_probe_hbm_read": [c_vp, c_i64, c_vp, c_vp],
    "pf_convert_f32": [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp],
    "pf_row_negentropy_f32": [c_vp, c_i64, c_i64, c_i64, c_dbl, c_vp, c_vp],
    "pf_dense_kl_f32": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_dbl, c_dbl, c_i64,
                        c_i64, c_vp, c_vp, c_i64, c_vp, c_dbl, c_vp, c_vp, c_vp],
    "pf_dense_tv_f32": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_dbl, c_dbl, c_i64, c_i64, c_vp,
                        c_vp, c_i64, c_vp, c_vp, c_vp],
    "pf_mask_compare_f64": [c_vp, c_vp, c_i64, c_dbl, c_vp, c_vp],
    # struct arguments (pf_mesh_t*, pf_paths_t*) are passed as addresses
    "pf_trace_batch_f64": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp],
    "pf_trace_fields_f64": [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp],
    "pf_triangle_gradient_f64": [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp],
    "pf_edge_descent_batch_f64": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp],
    "pf_local_minima_f64": [c_vp, c_vp, c_i64, c_vp, c_vp],
    "pf_np_hypot_f64": [c_vp, c_vp, c_i64, c_vp, c_vp],
    "pf_mesh_geometry_f64": [c_vp, c_vp, c_vp],
    "pf_mesh_pack_f64": [c_vp, c_vp, c_vp],
    "pf_format_lines": [c_vp, c_i64, c_int, c_i64, c_vp, c_vp, c_vp, c_vp],
    "pf_pack_lines": [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp],
    "pf_polyline_arc_f64": [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp],
    "pf_polyline_resample_f64": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp],
    "pf_hausdorff_pairs_f64": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                               c_i64, c_vp, c_vp],
}
# host-side symbolic plans (nd_plan.cpp): host pointers, opaque handle
_SIGS.update({
    "pf_nd_plan_build": [c_i64, c_vp, c_vp, c_vp, c_vp, c_int, c_int,
                         ctypes.POINTER(ctypes.c_void_p)],
    "pf_nd_plan_free": [c_vp],
    "pf_nd_plan_array": [c_vp, ctypes.c_char_p, c_vp],
    "pf_nd_plan_stats": [c_vp, c_vp],
    "pf_vertex_neighbors": [c_i64, c_i64, c_vp, c_vp, c_vp, ctypes.POINTER(ctypes.c_int64)],
    "pf_cotan_laplacian_f64": [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp,
                               c_vp],
    "pf_mf_factor_level": [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_int, c_vp, c_vp, c_vp],
    "pf_mf_inverse": [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp],
    "pf_mf_forward_level": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp,
                            c_i64, c_vp, c_vp, c_vp],
    "pf_mf_backward_level": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_int,
                             c_int, c_vp, c_i64, c_vp],
    "pf_poisson_residual_table": [c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp],
    "pf_poisson_residual": [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                            c_vp],
    "pf_poisson_finalize": [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_dbl, c_vp, c_vp,
                            c_vp, c_vp],
    "pf_poisson_residual_rows": [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                 c_vp, c_vp, c_vp],
    "pf_poisson_finalize_rows": [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                                 c_vp],
    # user generators (pf_jit.cu)
    "pf_user_compile": [ctypes.c_char_p, ctypes.c_char_p, c_int, ctypes.POINTER(ctypes.c_void_p)],
    "pf_user_cubin_size": [c_vp, ctypes.POINTER(ctypes.c_int64)],
    "pf_user_free": [c_vp],
    "pf_dense_user_f64": [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_dbl, c_int, c_i64, c_i64,
                          c_vp, c_vp, c_vp, c_vp],
    "pf_dense_user_at_f64": [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_dbl, c_int, c_i64, c_i64,
                             c_vp, c_i64, c_vp, c_vp],
    "pf_csr_user_f64": [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_dbl, c_i64, c_vp, c_i64,
                        c_vp, c_vp, c_vp],
    # NCCL plumbing (pf_nccl.cu): host id / handle pointers, device buffers
    "pf_nccl_load": [ctypes.c_char_p],
    "pf_nccl_version": [ctypes.POINTER(ctypes.c_int)],
    "pf_nccl_unique_id": [c_vp],
    "pf_nccl_comm_init": [c_int, c_vp, c_int, c_int, ctypes.POINTER(ctypes.c_void_p)],
    "pf_nccl_comm_destroy": [c_vp],
    "pf_nccl_broadcast": [c_vp, c_vp, c_i64, c_int, c_int, c_vp],
    "pf_nccl_all_gather": [c_vp, c_vp, c_vp, c_i64, c_int, c_vp],
    "pf_nccl_all_reduce": [c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_vp],
})
_RESTYPES = {"pf_last_error": ctypes.c_char_p, "pf_nd_plan_free": None,
             "pf_nd_plan_array": ctypes.c_int64, "pf_i8_tiled_bytes": ctypes.c_int64}



def load():
    """Load the shared library once; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeError(-100, f"{LIB_PATH.name} is not built; run "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
        return lib


def header_symbols() -> list[str]:
    """Every function declared in include/pathfield_b200.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char \*)\s*(pf_\w+)\s*\(", text, re.M)))


def symbols() -> list[str]:
    lib = load()
    return [s for s in header_symbols() if hasattr(lib, s)]


_fns: dict = {}


def call(name: str, *args) -> None:
    """Invoke an entry point; raise NativeError with pf_last_error() on failure."""
    fn = _fns.get(name)
    if fn is None:
        fn = _fns[name] = getattr(load(), name)
    rc = fn(*args)
    if rc != 0:
        msg = load().pf_last_error().decode(errors="replace")
        raise NativeError(rc, f"{name}: {msg}")


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else t.data_ptr()
