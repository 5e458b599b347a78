"""ctypes binding of libsmcl_gpu.so (include/smcl_gpu.h).

The shared library is built in-tree by ``make`` (``__graft_entry__.build()``).
There is no fallback: if the library is missing this module raises, so no
product path can silently run on the CPU.
"""
import ctypes as C
import os

from .abi import (SmclCloud, SmclComm, SmclConfig, SmclCorridorSpec, SmclFrameResult, SmclNeighborStats, SmclOdom,
                  SmclParticlesView, SmclSensorSpec, SmclStepProfile)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsmcl_gpu.so")

# Every symbol the header declares (checked by tests/test_abi.py).
_d, _i32, _i64, _u64, _int = C.c_double, C.c_int32, C.c_int64, C.c_uint64, C.c_int
_P = C.POINTER
SIGNATURES = {
    "smcl_abi_version": (_int, []),
    "smcl_last_error": (C.c_char_p, []),
    "smcl_config_default": (None, [_P(SmclConfig)]),
    "smcl_device_count": (_int, [_P(_int)]),
    "smcl_create": (_int, [_P(SmclCloud), _P(SmclConfig), _int, _P(C.c_void_p)]),
    "smcl_create_sharded": (_int, [_P(SmclCloud), _P(SmclConfig), _int, _P(SmclComm), _P(C.c_void_p)]),
    "smcl_comm_loopback_create": (_int, [_i32, _P(SmclComm)]),
    "smcl_comm_loopback_destroy": (None, [_P(SmclComm)]),
    "smcl_nccl_get_unique_id": (_int, [_P(C.c_uint8)]),
    "smcl_comm_nccl_create": (_int, [_P(C.c_uint8), _i32, _i32, _P(SmclComm)]),
    "smcl_comm_nccl_destroy": (None, [_P(SmclComm)]),
    "smcl_destroy": (_int, [C.c_void_p]),
    "smcl_init_uniform": (_int, [C.c_void_p, _P(_d)]),
    "smcl_init_uniform_seeded": (_int, [C.c_void_p, _i64, _P(_d), _int, _u64]),
    "smcl_step": (_int, [C.c_void_p, _P(SmclCloud), _P(SmclOdom), _P(SmclFrameResult)]),
    "smcl_scan_upload": (_int, [C.c_void_p, _int, _P(SmclCloud)]),
    "smcl_step_slot": (_int, [C.c_void_p, _int, _P(SmclOdom), _P(SmclFrameResult)]),
    "smcl_scan_prepare": (_int, [C.c_void_p, _int, _P(_d), _i64]),
    "smcl_scan_prepare_async": (_int, [C.c_void_p, _int, _P(_d), _i64]),
    "smcl_scan_get": (_int, [C.c_void_p, _int, _P(_d), _P(_d), _P(_i64)]),
    "smcl_step_points": (_int, [C.c_void_p, _P(_d), _i64, _P(SmclOdom), _P(SmclFrameResult)]),
    "smcl_last_step_profile": (_int, [C.c_void_p, _P(SmclStepProfile)]),
    "smcl_last_step_counts": (_int, [C.c_void_p, _P(SmclStepProfile)]),
    "smcl_timer_start": (_int, [C.c_void_p]),
    "smcl_timer_stop": (_int, [C.c_void_p, _P(_d)]),
    "smcl_frame_index": (_i64, [C.c_void_p]),
    "smcl_num_particles": (_i64, [C.c_void_p]),
    "smcl_get_particles": (_int, [C.c_void_p, _P(SmclParticlesView)]),
    "smcl_set_particles": (_int, [C.c_void_p, _P(SmclParticlesView)]),
    "smcl_get_nnf": (_int, [C.c_void_p, _P(_i32), _P(_d), _P(_d), _P(_i32)]),
    "smcl_predict": (_int, [C.c_void_p, _P(_d), _P(_d), _u64]),
    "smcl_update_neighbors": (_int, [C.c_void_p, _u64, _P(_d), _P(SmclNeighborStats)]),
    "smcl_evaluate_all": (_int, [C.c_void_p, _P(SmclCloud), _P(_d), _P(_d), _P(_i32), _P(_d), _P(_d)]),
    "smcl_evaluate_likelihoods": (_int, [C.c_void_p, _P(SmclCloud), _P(_d), _P(_i32)]),
    "smcl_compute_phis": (_int, [C.c_void_p, _P(_d), _P(_d)]),
    "smcl_apply_updates": (_int, [C.c_void_p, _P(_d)]),
    "smcl_bayes_update": (_int, [C.c_void_p, _P(_d), _P(_i32), _d, _d, _P(_i32)]),
    "smcl_normalize_log_post": (_int, [C.c_void_p, _d]),
    "smcl_smooth": (_int, [C.c_void_p, _i32, _d]),
    "smcl_representative": (_int, [C.c_void_p, _P(_i64), _P(_d), _P(_d)]),
    "smcl_se3_exp_batch": (_int, [_P(_d), _i64, _P(_d)]),
    "smcl_se3_log_batch": (_int, [_P(_d), _i64, _P(_d)]),
    "smcl_kernel_batch": (_int, [_P(_d), _P(_d), _i64, _d, _d, _P(_d)]),
    "smcl_lsh_hash_batch": (_int, [_P(_d), _i64, _P(_d), _P(_d), _d, _d, _d, _P(_u64)]),
    "smcl_solve_step_batch": (_int, [_P(_d), _P(_d), _P(_d), _i64, _d, _d, _P(_d)]),
    "smcl_estimate_covariances": (_int, [_P(_d), _i64, _int, _d, _P(_d)]),
    "smcl_downsample_to": (_int, [_P(_d), _i64, _i64, _d, _P(_d), _P(_i64)]),
    "smcl_make_scan_cloud": (_int, [_P(_d), _i64, _P(SmclConfig), _P(_d), _P(_d), _P(_i64)]),
    "smcl_build_nnf": (_int, [_P(SmclCloud), _d, _d, _d, _P(_i32), _P(_d), _P(_i32)]),
    "smcl_sim_default_corridor": (None, [_P(SmclCorridorSpec)]),
    "smcl_sim_default_sensor": (None, [_P(SmclSensorSpec)]),
    "smcl_sim_corridor_world": (_int, [_P(SmclCorridorSpec), _P(_d), _i32, _P(_i32)]),
    "smcl_sim_box_room": (_int, [_P(_d), _P(_d), _i32, _P(_i32)]),
    "smcl_sim_sample_world": (_int, [_P(_d), _i32, _d, _u64, _int, _d, _P(_d), _P(_d), _P(_i64)]),
    "smcl_sim_scan": (_int, [_P(_d), _i32, _P(_d), _P(SmclSensorSpec), _P(_u64), _P(_d), _P(_i64)]),
}

_lib = None


class SmclError(RuntimeError):
    """Error returned by the C ABI (SMCL_ERUNTIME / SMCL_ECUDA / SMCL_ENCCL)."""


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a extension first (make / __graft_entry__.build()). "
                "There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc):
    """Map an SMCL_E* code to the exception type the reference would throw."""
    if rc == 0:
        return
    msg = lib().smcl_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)  # std::invalid_argument
    if rc == 3:
        raise RuntimeError(f"logic_error: {msg}")  # std::logic_error
    raise SmclError(f"[smcl rc={rc}] {msg}")
