"""ctypes loader for the in-tree C ABI library libvrg.so (include/vrg.h).

The product path has no CPU fallback: if the library is missing or fails to load, every call
raises.  `load()` loads the .so on first use.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VRG_LIB_PATH", os.path.join(HERE, "libvrg.so"))  # override: experiments only
HEADER = os.path.join(os.path.dirname(HERE), "include", "vrg.h")

VRG_OK, VRG_INVALID_ARGUMENT, VRG_BLOWUP, VRG_RUNTIME_ERROR, VRG_NOT_SUPPORTED = 0, 1, 2, 3, 4

_lib = None

# Argument kinds of every exported symbol: p = pointer, i = int, d = double, u = u64.
_SIG = {
    "vrg_version": ("", C.c_char_p),
    "vrg_ctx_create": ("ipp", C.c_int),
    "vrg_ctx_destroy": ("p", None),
    "vrg_ctx_stream": ("p", C.c_void_p),
    "vrg_set_penalty_weight": ("pd", C.c_int),
    "vrg_set_scheme": ("pi", C.c_int),
    "vrg_last_error": ("p", C.c_char_p),
    "vrg_sync": ("p", C.c_int),
    "vrg_malloc": ("pup", C.c_int),
    "vrg_free": ("pp", C.c_int),
    "vrg_host_alloc": ("pup", C.c_int),
    "vrg_host_free": ("pp", C.c_int),
    "vrg_copy_h2d": ("pppu", C.c_int),
    "vrg_copy_d2h": ("pppu", C.c_int),
    "vrg_counters": ("ppp", C.c_int),
    "vrg_counters_reset": ("p", C.c_int),
    "vrg_launch_count": ("pp", C.c_int),
    "vrg_profile": ("pi", C.c_int),
    "vrg_profile_dump": ("ppi", C.c_int),
    "vrg_dot": ("piipppp" + "p", C.c_int),
    "vrg_norm_linf": ("piippp", C.c_int),
    "vrg_axpy": ("pudpp", C.c_int),
    "vrg_prefilter": ("piipp", C.c_int),
    "vrg_evaluate": ("piipppp", C.c_int),
    "vrg_derive_steps": ("piippdp", C.c_int),
    "vrg_trace": ("piippdipp", C.c_int),
    "vrg_solver_create": ("piippip", C.c_int),
    "vrg_solver_create_ex": ("piippiip", C.c_int),
    "vrg_solver_stages": ("pp", C.c_int),
    "vrg_solver_destroy": ("p", None),
    "vrg_solver_state": ("ppp", C.c_int),
    "vrg_solver_adjoint": ("ppp", C.c_int),
    "vrg_solver_state_final": ("ppp", C.c_int),
    "vrg_solver_adjoint_final": ("ppp", C.c_int),
    "vrg_solver_incstate": ("ppppp", C.c_int),
    "vrg_solver_incadjoint": ("pppppip", C.c_int),
    "vrg_solver_jacobian": ("pp", C.c_int),
    "vrg_solver_departure": ("pipp", C.c_int),
    "vrg_gradient": ("piippp", C.c_int),
    "vrg_apply_helmholtz": ("piipp", C.c_int),
    "vrg_body_force": ("piiipppp", C.c_int),
    "vrg_divergence": ("piippp", C.c_int),
    "vrg_apply_reg": ("piiidpppp", C.c_int),
    "vrg_apply_inv_reg": ("piiiddpppp", C.c_int),
    "vrg_project_div_free": ("piipppp", C.c_int),
    "vrg_resample": ("piipiip", C.c_int),
    "vrg_cutoff": ("piipip", C.c_int),
    "vrg_gaussian_smooth": ("piipdp", C.c_int),
    "vrg_hess_create": ("piippppidiiipp", C.c_int),
    "vrg_hess_create_ex": ("piipppppiiippp", C.c_int),
    "vrg_hess_destroy": ("p", None),
    "vrg_hess_create_batch": ("piiippppidiip", C.c_int),
    "vrg_hess_apply": ("ppppp", C.c_int),
    "vrg_hess_apply_data": ("ppppp", C.c_int),
    "vrg_hess_apply_split": ("ppppp", C.c_int),
    "vrg_hess_apply_host": ("ppppp", C.c_int),
    "vrg_hess_apply_host_batch": ("pipppp", C.c_int),
    "vrg_hess_apply_batch": ("pipppp", C.c_int),
    "vrg_hess_graph_info": ("pp", C.c_int),
    "vrg_hess_state": ("pp", C.c_int),
    "vrg_hess_bench_kernel": ("piip", C.c_int),
    "vrg_hess_band_path": ("pp", C.c_int),
    "vrg_band_mapping": ("i", C.c_int),
    "vrg_newton_solve_batch": ("piiippidipppppppipp", C.c_int),
    "vrg_hess_buffers": ("pp", C.c_int),
    "vrg_prefilter_rows": ("piippp", C.c_int),
    "vrg_slab_cols": ("piipp", C.c_int),
    "vrg_slab_step": ("piiiiiippppiddpppp", C.c_int),
    "vrg_evaluate_gradient": ("piippppidiippp", C.c_int),
    "vrg_evaluate_gradient_ex": ("piipppppiippppppppp", C.c_int),
    "vrg_evaluate_objective_ex": ("piipppppiippp", C.c_int),
    "vrg_evaluate_objective": ("piippppidiip", C.c_int),
    "vrg_random_bandlimited_field": ("piiup", C.c_int),
    "vrg_coarse_create": ("piippppididp", C.c_int),
    "vrg_coarse_destroy": ("p", None),
    "vrg_coarse_info": ("pppp", C.c_int),
    "vrg_coarse_apply_split": ("ppppp", C.c_int),
    "vrg_two_level_apply": ("pppiiddddppp", C.c_int),
    "vrg_estimate_eigs": ("piippppididupp", C.c_int),
    "vrg_solve_kkt": ("pppdippppppdppp", C.c_int),
    "vrg_newton_solve": ("piippidipppppppip", C.c_int),
    "vrg_newton_solve_ex": ("piippppppppip", C.c_int),
    "vrg_set_fine_operator": ("pppp", C.c_int),
    "vrg_set_external_ops": ("pp", C.c_int),
}

_KIND = {"p": C.c_void_p, "i": C.c_int, "d": C.c_double, "u": C.c_ulonglong}


def header_symbols():
    """Names of all functions declared in include/vrg.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|void\*|void|const char\*)\s+(vrg_\w+)\s*\(", text, re.M)))


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make` (the CUDA path has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (kinds, res) in _SIG.items():
            fn = getattr(lib, name)
            fn.argtypes = [_KIND[k] for k in kinds]
            fn.restype = res
        _lib = lib
    return _lib
