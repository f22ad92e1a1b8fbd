"""ctypes declarations of the include/splbcu.h C-ABI (structs and the
signature of every exported symbol).

Pure declarations: importing this module loads no shared library, so the
test oracles (tests/impls.py) and the reference arm of bench.py can bind the
same C-ABI implemented by other libraries without mapping libsplbcu.so.
"""
from __future__ import annotations

import ctypes as C

c_int = C.c_int32
c_u8p = C.POINTER(C.c_uint8)
c_u16p = C.POINTER(C.c_uint16)
c_u32p = C.POINTER(C.c_uint32)
c_u64p = C.POINTER(C.c_uint64)
c_i32p = C.POINTER(C.c_int32)
c_dp = C.POINTER(C.c_double)


class Iolet(C.Structure):
    _fields_ = [("kind", C.c_int32), ("center", C.c_double * 3), ("normal", C.c_double * 3),
                ("radius", C.c_double)]


class BC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("times", c_dp), ("values", c_dp), ("n_nodes", C.c_uint32),
                ("period", C.c_double)]


class Params(C.Structure):
    _fields_ = [("tau", C.c_double), ("rho0", C.c_double), ("dt_s", C.c_double),
                ("layout", C.c_int32), ("scheme", C.c_int32), ("sequence", C.c_int32),
                ("workers", C.c_int32), ("capture_period", C.c_uint64),
                ("observe_iolets", C.c_int32), ("exchange_timeout_s", C.c_double),
                ("n_devices", C.c_int32), ("device_ids", c_i32p), ("halo_mode", C.c_int32),
                ("storage", C.c_int32)]


# (name, restype, argtypes) for every symbol include/splbcu.h declares.
_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
SIGNATURES = [
    ("splbcu_last_error", C.c_char_p, []),
    ("splbcu_version", C.c_char_p, []),
    ("splbcu_params_default", None, [C.POINTER(Params)]),
    ("splbcu_equilibrium", None, [C.c_double, c_dp, c_dp]),
    ("splbcu_moments", c_int, [c_dp, c_dp, c_dp]),
    ("splbcu_bgk_collide", c_int, [c_dp, C.c_double, c_dp]),
    ("splbcu_timetable_at", c_int, [c_dp, c_dp, C.c_uint32, C.c_double, C.c_double, c_dp]),
    ("splbcu_iolet_weight", C.c_double, [C.POINTER(Iolet), c_i32p]),
    ("splbcu_domain_classify", c_int, [c_i32p, C.c_uint64, C.POINTER(Iolet), C.c_uint32, C.c_double, _PP]),
    ("splbcu_domain_build_pipe", c_int, [c_int, c_int, C.c_double, _PP]),
    ("splbcu_domain_build_bifurcation", c_int, [c_int, c_int, c_int, c_int, C.c_double, _PP]),
    ("splbcu_domain_build_tree", c_int, [c_int, c_int, c_int, C.c_double, C.c_double, C.c_double, _PP]),
    ("splbcu_domain_build_channel", c_int, [c_int, c_int, c_int, C.c_double, _PP]),
    ("splbcu_domain_from_arrays", c_int, [C.c_uint64, c_i32p, c_u8p, c_u8p, c_u16p, C.POINTER(Iolet),
                                          C.c_uint32, c_u64p, C.c_double, _PP]),
    ("splbcu_domain_validate", c_int, [_P]),
    ("splbcu_domain_read", c_int, [C.c_char_p, _PP]),
    ("splbcu_domain_write", c_int, [_P, C.c_char_p]),
    ("splbcu_domain_n_sites", C.c_uint64, [_P]),
    ("splbcu_domain_n_iolets", C.c_uint32, [_P]),
    ("splbcu_domain_voxel_size", C.c_double, [_P]),
    ("splbcu_domain_export", c_int, [_P, c_i32p, c_u8p, c_u8p, c_u16p, C.POINTER(Iolet), c_u64p]),
    ("splbcu_domain_free", None, [_P]),
    ("splbcu_source_pipe", c_int, [c_int, c_int, C.c_double, _PP]),
    ("splbcu_source_bifurcation", c_int, [c_int, c_int, c_int, c_int, C.c_double, _PP]),
    ("splbcu_source_tree", c_int, [c_int, c_int, c_int, C.c_double, C.c_double, C.c_double, _PP]),
    ("splbcu_source_channel", c_int, [c_int, c_int, c_int, C.c_double, _PP]),
    ("splbcu_source_build", c_int, [_P, _PP]),
    ("splbcu_source_window", c_int, [_P, c_int, c_int, c_i32p, _PP, _PP]),
    ("splbcu_window_info", c_int, [_P, c_u64p, c_i32p, c_i32p, c_u64p]),
    ("splbcu_source_free", None, [_P]),
    ("splbcu_partition_create", c_int, [_P, c_int, _PP]),
    ("splbcu_partition_global", c_int, [_P, c_i32p, c_u32p]),
    ("splbcu_partition_part_shape", c_int, [_P, c_int, c_u32p, c_u32p, c_u32p]),
    ("splbcu_partition_part", c_int, [_P, c_int, c_u32p, c_u64p, c_u64p, c_i32p]),
    ("splbcu_partition_imbalance", C.c_double, [_P]),
    ("splbcu_partition_free", None, [_P]),
    ("splbcu_sim_create", c_int, [_P, C.POINTER(BC), C.c_uint32, C.POINTER(Params), _PP]),
    ("splbcu_nccl_unique_id", c_int, [c_u8p]),
    ("splbcu_sim_create_dist", c_int, [_P, C.POINTER(BC), C.c_uint32, C.POINTER(Params), c_int, c_int,
                                       c_u8p, _PP]),
    ("splbcu_sim_create_dist_source", c_int, [_P, C.POINTER(BC), C.c_uint32, C.POINTER(Params), c_int, c_int,
                                              c_u8p, _PP]),
    ("splbcu_sim_slab_local", c_int, [_P]),
    ("splbcu_sim_n_sites", C.c_uint64, [_P]),
    ("splbcu_sim_run", c_int, [_P, C.c_uint64]),
    ("splbcu_sim_steps_run", C.c_uint64, [_P]),
    ("splbcu_sim_step_loop_seconds", C.c_double, [_P]),
    ("splbcu_sim_device_loop_seconds", C.c_double, [_P]),
    ("splbcu_sim_snapshot", c_int, [_P, c_dp]),
    ("splbcu_sim_n_workers", c_int, [_P]),
    ("splbcu_sim_worker_is_local", c_int, [_P, c_int]),
    ("splbcu_sim_store_shape", c_int, [_P, c_int, c_u32p, c_u32p]),
    ("splbcu_sim_get_f", c_int, [_P, c_int, c_int, c_dp]),
    ("splbcu_sim_set_f", c_int, [_P, c_int, c_int, c_dp]),
    ("splbcu_sim_map_shape", c_int, [_P, c_int, c_u32p, c_u32p, c_u32p]),
    ("splbcu_sim_export_map", c_int, [_P, c_int, c_u32p, c_u8p, c_u16p, c_u32p, c_u32p, c_u8p, c_i32p,
                                      c_u32p, c_u32p]),
    ("splbcu_sim_export_sources", c_int, [_P, c_int, c_u32p, c_u8p, c_u16p]),
    ("splbcu_sim_partition", _P, [_P]),
    ("splbcu_sim_n_captures", C.c_uint64, [_P]),
    ("splbcu_sim_capture", c_int, [_P, C.c_uint64, c_u64p, c_dp]),
    ("splbcu_sim_series_rows", C.c_uint64, [_P]),
    ("splbcu_sim_series", c_int, [_P, C.c_uint32, c_dp, c_dp, c_dp]),
    ("splbcu_sim_write_snapshots", c_int, [_P, C.c_char_p]),
    ("splbcu_sim_series_csv", c_int, [_P, C.c_double, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("splbcu_sim_set_kernel_timing", c_int, [_P, c_int]),
    ("splbcu_sim_kernel_stats", c_int, [_P, c_dp, c_u64p, c_u64p]),
    ("splbcu_sim_launch_count", C.c_uint64, [_P]),
    ("splbcu_sim_bulk_kernel", C.c_int32, [_P]),
    ("splbcu_sim_series_d2h_bytes", C.c_uint64, [_P]),
    ("splbcu_sim_destroy", None, [_P]),
]
