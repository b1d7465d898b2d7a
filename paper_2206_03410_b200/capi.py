"""ctypes binding of include/nrr_cuda.h (libnrr_b200.so).

The library is the product: every call goes to the sm_100a kernels through
the C ABI. There is no CPU fallback — if the shared library is missing or no
B200 is visible the calls raise.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# NRR_LIB_PATH: an alternative build of this library (A/B experiments)
LIB_PATH = os.environ.get("NRR_LIB_PATH") or os.path.join(_HERE, "libnrr_b200.so")

i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class NrrError(RuntimeError):
    code = 5


class IoError(NrrError):
    code = 2


class NumericalError(NrrError):
    code = 3


class ConfigError(NrrError):
    code = 4


class CudaError(NrrError):
    code = 5


_ERRORS = {2: IoError, 3: NumericalError, 4: ConfigError, 5: CudaError}


class ProblemView(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("source", f64p), ("src_avg_edge_length", C.c_double),
        ("m", C.c_int32), ("target", f64p),
        ("node_count", C.c_int32), ("node_positions", f64p),
        ("edge_count", C.c_int32), ("edges", i32p),
        ("infl_offsets", i32p), ("infl_nodes", i32p), ("infl_weights", f64p),
        ("pair_count", C.c_int32), ("reg_pairs", i32p), ("reg_weights", f64p),
    ]


class SolverConfig(C.Structure):
    _fields_ = [
        ("k_alpha", C.c_double), ("k_beta", C.c_double), ("eps", C.c_double),
        ("i_max", C.c_int32), ("aa_window", C.c_int32),
        ("nu_a_init", C.c_double), ("nu_a_min", C.c_double), ("nu_r_init", C.c_double),
        ("nu_r_floor", C.c_double),
        ("landmark_count", C.c_int32), ("landmark_index", i32p), ("landmark_pos", f64p),
    ]


class IterationRecord(C.Structure):
    _fields_ = [("e_total", C.c_double), ("e_align", C.c_double), ("e_reg", C.c_double),
                ("e_rot", C.c_double), ("e_landmark", C.c_double), ("max_disp", C.c_double),
                ("aa_accepted", C.c_int32), ("stage", C.c_int32)]


class StageRecord(C.Structure):
    _fields_ = [("nu_a", C.c_double), ("nu_r", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("reverts", C.c_int32), ("converged", C.c_int32), ("first_iteration", C.c_int32),
                ("iteration_count", C.c_int32)]


class PassRecord(C.Structure):
    _fields_ = [("e_total", C.c_double), ("stage", C.c_int32), ("reverted", C.c_int32)]


class ReportSummary(C.Structure):
    _fields_ = [("stage_count", C.c_int32), ("total_iterations", C.c_int32),
                ("degenerate_rotations", C.c_int32), ("alpha_forced_zero", C.c_int32),
                ("total_passes", C.c_int32), ("linear_iterations", C.c_int32),
                ("solve_seconds", C.c_double), ("setup_seconds", C.c_double), ("loop_seconds", C.c_double)]


class PassTrace(C.Structure):
    _fields_ = [("e_align", C.c_double), ("e_reg", C.c_double), ("e_rot", C.c_double), ("e_total", C.c_double),
                ("e_landmark", C.c_double), ("max_disp", C.c_double), ("stage", C.c_int32),
                ("reverted", C.c_int32), ("pcg_iterations", C.c_int32), ("accepted_index", C.c_int32)]


class SolveOptions(C.Structure):
    _fields_ = [("pcg_rtol", C.c_double), ("pcg_max_iter", C.c_int32), ("record_passes", C.c_int32),
                ("max_ctas", C.c_int32)]


_SIGS = {
    "nrr_last_error": (C.c_char_p, []),
    "nrr_device_info": (C.c_int, [C.c_int, C.c_char_p, C.c_int32, i32p]),
    "nrr_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "nrr_ctx_destroy": (None, [C.c_void_p]),
    "nrr_ctx_set_options": (C.c_int, [C.c_void_p, C.POINTER(SolveOptions)]),
    "nrr_ctx_set_target": (C.c_int, [C.c_void_p, f64p, C.c_int32]),
    "nrr_ctx_set_problem": (C.c_int, [C.c_void_p, C.POINTER(ProblemView)]),
    "nrr_ctx_register": (C.c_int, [C.c_void_p, C.POINTER(SolverConfig), f64p, f64p]),
    "nrr_ctx_begin": (C.c_int, [C.c_void_p, C.POINTER(SolverConfig)]),
    "nrr_ctx_iterate": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, i32p, i32p, f64p]),
    "nrr_ctx_finish": (C.c_int, [C.c_void_p, f64p, f64p]),
    "nrr_register": (C.c_int, [C.c_void_p, C.POINTER(ProblemView), C.POINTER(SolverConfig), f64p, f64p]),
    "nrr_ctx_report": (C.c_int, [C.c_void_p, C.POINTER(ReportSummary), C.POINTER(StageRecord), C.c_int32,
                                 C.POINTER(IterationRecord), C.c_int32, C.POINTER(PassRecord), C.c_int32, i32p]),
    "nrr_ctx_trace_count": (C.c_int, [C.c_void_p, i32p]),
    "nrr_ctx_trace": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(PassTrace), f64p, f64p, i32p]),
    "nrr_nearest": (C.c_int, [C.c_void_p, f64p, C.c_int32, i32p, f64p]),
    "nrr_nearest_from": (C.c_int, [C.c_void_p, f64p, C.c_int32, i32p, i32p, f64p]),
    "nrr_deform": (C.c_int, [C.c_void_p, f64p, f64p]),
    "nrr_project_rotations": (C.c_int, [C.c_void_p, f64p, C.c_int32, f64p, i32p]),
    "nrr_step": (C.c_int, [C.c_void_p, f64p, f64p, C.c_double, C.POINTER(SolverConfig), i32p, f64p, f64p,
                           f64p, f64p, f64p]),
    "nrr_comm_unique_id": (C.c_int, [C.c_void_p]),
    "nrr_ctx_set_comm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]),
    "nrr_ctx_set_shard": (C.c_int, [C.c_void_p, C.c_int32]),
    "nrr_local_group_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "nrr_local_group_destroy": (None, [C.c_void_p]),
    "nrr_ctx_set_local_comm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "nrr_assemble": (C.c_int, [C.c_void_p, f64p, f64p, f64p, f64p, C.c_double, C.c_double,
                               C.POINTER(SolverConfig), f64p, f64p]),
    "nrr_solve": (C.c_int, [C.c_void_p, f64p, f64p, f64p, f64p]),
    "nrr_anderson_combine": (C.c_int, [C.c_void_p, f64p, f64p, C.c_int32, C.c_int32, C.c_int32, f64p, i32p]),
    "nrr_init_parameters": (C.c_int, [C.c_void_p, C.POINTER(SolverConfig), f64p]),
    "nrr_ctx_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), f64p, i32p]),
    "nrr_ctx_comm_ms": (C.c_int, [C.c_void_p, f64p]),
    "nrr_ctx_enable_timing": (C.c_int, [C.c_void_p, C.c_int32]),
    "nrr_debug_solver_plan": (C.c_int, [C.POINTER(ProblemView), C.c_int32, C.c_int64, C.POINTER(C.c_int64)]),
    "nrr_debug_pcg_partition": (C.c_int, [C.POINTER(ProblemView), C.c_int32, C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "nrr_edges_from_faces": (C.c_int, [i32p, C.c_int32, C.c_int32, i32p, C.c_int32, i32p]),
    "nrr_knn_edges": (C.c_int, [f64p, C.c_int32, C.c_int32, i32p, C.c_int32, i32p]),
    "nrr_avg_edge_length": (C.c_int, [f64p, C.c_int32, i32p, C.c_int32, f64p]),
    "nrr_normalize_pair": (C.c_int, [f64p, C.c_int32, f64p, C.c_int32, f64p]),
    "nrr_build_graph": (C.c_int, [f64p, C.c_int32, i32p, C.c_int32, C.c_double, C.POINTER(C.c_void_p)]),
    "nrr_build_graph_gpu": (C.c_int, [C.c_int32, f64p, C.c_int32, i32p, C.c_int32, C.c_double, C.POINTER(C.c_void_p),
                                      i32p]),
    "nrr_knn_edges_gpu": (C.c_int, [C.c_int32, f64p, C.c_int32, C.c_int32, i32p, C.c_int32, i32p]),
    "nrr_device_count": (C.c_int, [i32p]),
    "nrr_project_rotations_sigma": (C.c_int, [C.c_void_p, f64p, C.c_int32, f64p, f64p, i32p]),
    "nrr_energy_terms": (C.c_int, [C.c_void_p, C.c_void_p, f64p, f64p, f64p]),
    "nrr_limited_geodesic": (C.c_int, [f64p, C.c_int32, i32p, C.c_int32, C.c_int32, C.c_double, i32p, f64p,
                                       C.c_int32, i32p]),
    "nrr_graph_counts": (None, [C.c_void_p, i32p, i32p, i32p, i32p]),
    "nrr_graph_export": (None, [C.c_void_p, i32p, f64p, i32p, i32p, i32p, f64p, f64p, i32p, f64p]),
    "nrr_graph_free": (None, [C.c_void_p]),
    "nrr_synth_config": (C.c_int, [C.c_int32, C.c_uint64, C.c_double, i32p, i32p, i32p, f64p, i32p, f64p]),
}

EXPORTED = sorted(_SIGS)

_lib = None


def load():
    """Load libnrr_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libnrr_b200.so not built: run `python -m paper_2206_03410_b200.build`")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc):
    if rc != 0:
        msg = load().nrr_last_error().decode()
        raise _ERRORS.get(rc, NrrError)(msg)


def ptr(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def d(a):
    return ptr(a, f64p)


def i(a):
    return ptr(a, i32p)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)
