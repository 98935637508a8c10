"""ctypes description of the C-ABI in include/rs.h.

The same plain-C surface is exported by three libraries:
  librs_b200.so               the product (prefix ``rs_``, takes an rs_ctx*)
  oracle/_ref/librollsim_ref_capi.so   the reference itself (prefix ``ref_``)
  oracle/build/liboracle_port.so       the C restatement (prefix ``orc_``)
The oracle libraries are test infrastructure and are bound in tests/.
"""
import ctypes as C

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
vp = C.c_void_p
P_i32, P_i64, P_u64, P_f64 = (C.POINTER(t) for t in (i32, i64, u64, f64))


class RsProfile(C.Structure):
    _fields_ = [
        ("batch_knots", P_f64), ("nb", i32),
        ("context_knots", P_f64), ("nc", i32),
        ("tpot_grid", P_f64), ("rho", f64),
    ]


class RsScaleOut(C.Structure):
    _fields_ = [
        ("n_star", i32),
        ("t_total", P_f64), ("t_penalty", P_f64), ("cost", P_f64),
        ("t_norm", P_f64), ("c_norm", P_f64), ("score", P_f64),
        ("idle_slot_ticks", P_i64), ("order", P_i32),
        ("actor_times", P_f64), ("group_times", P_f64),
        ("lpt_makespan", P_i64), ("lpt_idle", P_i64),
    ]


class RsScenarioSpec(C.Structure):
    _fields_ = [
        ("base_seed", u64), ("first_scenario", i64), ("n_scenarios", i32),
        ("count", i32), ("plen_mean", f64), ("plen_sigma", f64),
        ("plen_min", i32), ("plen_max", i32), ("pred_scale", f64),
        ("pred_min", f64), ("pred_max", f64),
    ]


class RsSweepOut(C.Structure):
    _fields_ = [
        ("t_total", vp), ("cost", vp), ("idle_slot_ticks", vp),
        ("n_star", vp), ("nstar_hist", vp), ("sum_t", vp), ("sum_c", vp),
    ]


class RsTopology(C.Structure):
    _fields_ = [
        ("n_nodes", i32), ("node_gpus", P_i32),
        ("intra_node_bw", f64), ("inter_node_bw", f64), ("bw_matrix", P_f64),
        ("learner_node", i32), ("n_learner_gpus", i32), ("learner_gpus", P_i32),
    ]


class RsPlacementPenalty(C.Structure):
    _fields_ = [
        ("topology", C.POINTER(RsTopology)), ("model_bytes", f64),
        ("kv_bytes_per_token", f64), ("l_prefill_seconds", f64),
    ]


class RsNoiseModel(C.Structure):
    _fields_ = [("kind", i32), ("bucket_accuracy", f64), ("bucket_width", i32), ("seed", u64)]


P_prof = C.POINTER(RsProfile)
P_pen = C.POINTER(RsPlacementPenalty)
P_noise = C.POINTER(RsNoiseModel)

# name -> argtypes (without the leading ctx for rs_* compute calls)
PRODUCT_SIGS = {
    "rs_last_error": ([], C.c_char_p),
    "rs_abi_version": ([], C.c_int),
    "rs_ctx_create": ([C.c_int, C.POINTER(vp)], C.c_int),
    "rs_ctx_destroy": ([vp], C.c_int),
    "rs_ctx_set_stream": ([vp, vp], C.c_int),
    "rs_ctx_synchronize": ([vp], C.c_int),
    "rs_ctx_kernel_launches": ([vp, P_u64], C.c_int),
    "rs_ctx_enable_kernel_timing": ([vp, C.c_int], C.c_int),
    "rs_ctx_reset_kernel_timing": ([vp], C.c_int),
    "rs_ctx_kernel_time": ([vp, C.c_char_p, P_f64, P_u64], C.c_int),
    "rs_tpot_seconds": ([vp, P_prof, P_f64, P_f64, i64, P_f64], C.c_int),
    "rs_prefix_index_build": ([vp, P_i32, P_i64, i32, C.POINTER(vp)], C.c_int),
    "rs_prefix_index_build_device": ([vp, vp, vp, i32, C.POINTER(vp)], C.c_int),
    "rs_prefix_index_build_device_async": ([vp, vp, vp, i32, i32, vp, vp], C.c_int),
    "rs_prefix_index_free": ([vp], None),
    "rs_prefix_index_from_tables": ([i32, i32, i32, i64, P_i64, P_i64, P_i64, P_i64, P_i64,
                                     C.POINTER(vp)], C.c_int),
    "rs_prefix_index_info": ([vp, P_i32, P_i32, P_i32, P_i64], C.c_int),
    "rs_unique_prefix_count": ([vp, i32, P_i64], C.c_int),
    "rs_unique_prefix_tokens": ([vp, i32, P_i64], C.c_int),
    "rs_remainder_tokens": ([vp, i32, P_i64], C.c_int),
    "rs_prefix_index_tables": ([vp, P_i64, P_i64, P_i64, P_i64, P_i64], C.c_int),
    "rs_select_prefix_length": ([vp, i32, i32, i32, i32, P_i32, P_i32], C.c_int),
    "rs_dedup_savings": ([vp, i32, i32, P_i64, P_i64, P_f64], C.c_int),
    "rs_unique_prefix_count_among": ([vp, P_i32, P_i64, i32, i32, P_i64], C.c_int),
    "rs_dedup_map": ([vp, P_i32, P_i64, i32, i32, P_i32], C.c_int),
    "rs_block_hashes": ([vp, P_i32, P_i64, i32, i32, P_u64], C.c_int),
    "rs_rank_strings": ([vp, C.c_char_p, P_i64, i32, P_i32], C.c_int),
    "rs_assign": ([vp, P_f64, P_i32, i32, i32, P_i32, P_i32], C.c_int),
    "rs_integrate_decode_seconds": ([vp, P_i32, P_f64, i64, P_prof, P_f64], C.c_int),
    "rs_estimate_actor_time": ([vp, P_i32, P_f64, i32, P_prof, i32, P_f64], C.c_int),
    "rs_estimate_cost": ([vp, P_i32, P_f64, P_i32, P_i32, i32, P_prof, i32, P_f64, P_f64], C.c_int),
    "rs_scale": ([vp, P_f64, P_i32, P_i32, i32, P_prof, i32, i32, i32, f64, i32, P_f64,
                  C.POINTER(RsScaleOut)], C.c_int),
    "rs_scale_placed": ([vp, P_f64, P_i32, P_i32, i32, P_prof, i32, i32, i32, f64, i32, P_pen,
                         C.POINTER(RsScaleOut)], C.c_int),
    "rs_predict_lengths": ([vp, vp, vp, vp, i32, i32, f64, i32, P_noise, vp, vp, C.c_int, vp],
                           C.c_int),
    "rs_trace_csr_parse": ([vp, vp, i64, C.c_int, C.POINTER(vp)], C.c_int),
    "rs_trace_csr_parse_jsonl": ([vp, vp, i64, C.c_int, C.POINTER(vp)], C.c_int),
    "rs_trace_csr_info": ([vp, P_i32, P_i64, P_i64, P_i32, P_i32, P_i32], C.c_int),
    "rs_trace_csr_device": ([vp, C.POINTER(vp), C.POINTER(vp)], C.c_int),
    "rs_trace_csr_copy": ([vp, vp, vp, vp, vp, vp, vp], C.c_int),
    "rs_trace_csr_steps_info": ([vp, P_i32, P_i64], C.c_int),
    "rs_trace_csr_steps_device": ([vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)],
                                  C.c_int),
    "rs_trace_csr_steps_copy": ([vp, vp, vp, vp, vp, vp], C.c_int),
    "rs_trace_csr_free": ([vp], None),
    "rs_scale_select": ([vp, P_f64, P_f64, P_f64, i32, i32, f64, P_f64, P_f64, P_f64, P_i32], C.c_int),
    "rs_generate_scenarios": ([vp, C.POINTER(RsScenarioSpec), vp, vp, C.c_int], C.c_int),
    "rs_sweep": ([vp, C.POINTER(RsScenarioSpec), P_prof, i32, i32, i32, f64, i32,
                  C.POINTER(RsSweepOut), C.c_int], C.c_int),
    "rs_sweep_arrays": ([vp, vp, vp, i32, i32, P_prof, i32, i32, i32, f64, i32,
                         C.POINTER(RsSweepOut), C.c_int], C.c_int),
    "rs_sweep_select": ([P_f64, P_f64, i64, i32, i32, f64, P_i32], C.c_int),
    "rs_lpt": ([vp, P_f64, P_i32, i32, i32, i32, i32, P_i64, P_i64], C.c_int),
    "rs_comm_unique_id": ([vp], C.c_int),
    "rs_comm_init": ([vp, vp, i32, i32, C.POINTER(vp)], C.c_int),
    "rs_comm_destroy": ([vp], C.c_int),
    "rs_sweep_sharded": ([vp, vp, C.POINTER(RsScenarioSpec), P_prof, i32, i32, i32, f64, i32,
                          C.POINTER(RsSweepOut), C.c_int, P_i32], C.c_int),
    "rs_multi_create": ([P_i32, i32, C.POINTER(vp)], C.c_int),
    "rs_multi_size": ([vp, P_i32], C.c_int),
    "rs_multi_context": ([vp, i32, C.POINTER(vp)], C.c_int),
    "rs_multi_destroy": ([vp], C.c_int),
    "rs_multi_sweep": ([vp, C.POINTER(RsScenarioSpec), P_prof, i32, i32, i32, f64, i32,
                        C.POINTER(RsSweepOut), P_i32], C.c_int),
}

# Plain-C oracle surface shared by ref_* and orc_* (oracle/oracle.h).
ORACLE_SIGS = {
    "last_error": ([], C.c_char_p),
    "tpot_seconds": ([P_prof, P_f64, P_f64, i64, P_f64], C.c_int),
    "prefix_curves": ([P_i32, P_i64, i32, i32, P_i64, P_i64, P_i64, P_i64], C.c_int),
    "select_prefix_length": ([P_i32, P_i64, i32, i32, i32, i32, i32, P_i32, P_i32], C.c_int),
    "dedup_savings": ([P_i32, P_i64, i32, i32, i32, P_i64, P_i64, P_f64], C.c_int),
    "unique_prefix_count_among": ([P_i32, P_i64, i32, i32, P_i64], C.c_int),
    "assign": ([P_f64, P_i32, i32, i32, P_i32, P_i32], C.c_int),
    "integrate_decode_seconds": ([P_i32, P_f64, i64, P_prof, P_f64], C.c_int),
    "estimate_actor_time": ([P_i32, P_f64, i32, P_prof, i32, P_f64], C.c_int),
    "estimate_cost": ([P_i32, P_f64, P_i32, P_i32, i32, P_prof, i32, P_f64, P_f64], C.c_int),
    "scale": ([P_f64, P_i32, P_i32, i32, P_prof, i32, i32, i32, f64, i32, P_f64, P_i32,
               P_f64, P_f64, P_f64, P_f64, P_f64, P_f64, P_i32, P_f64], C.c_int),
    "sweep_arrays": ([P_f64, P_i32, i32, i32, P_prof, i32, i32, i32, f64, i32, i32,
                      P_f64, P_f64, P_i32], C.c_int),
    "scale_placed": ([P_f64, P_i32, P_i32, i32, P_prof, i32, i32, i32, f64, i32, P_pen, P_i32,
                      P_f64, P_f64, P_f64, P_f64, P_f64, P_f64, P_i32, P_f64], C.c_int),
    "predict_lengths": ([P_f64, P_i32, P_i32, i32, i32, f64, i32, P_noise, C.c_char_p, P_i64,
                         P_f64], C.c_int),
}

REF_ONLY_SIGS = {
    "ref_trace_prompts": ([vp, i64, P_i64, vp, vp, vp, vp, vp], C.c_int),
    "ref_trace_steps": ([vp, i64, P_i64, vp, vp, vp, vp], C.c_int),
    "ref_trace_set_format": ([C.c_int], None),
    "ref_trace_convert": ([vp, i64, C.c_int, C.c_int, vp, i64, P_i64], C.c_int),
}

PORT_ONLY_SIGS = {
    "orc_generate_scenarios": ([C.POINTER(RsScenarioSpec), P_f64, P_i32], C.c_int),
    "orc_scale_idle": ([P_f64, P_i32, i32, i32, i32, i32, P_i64], C.c_int),
    "orc_dedup_map": ([P_i32, P_i64, i32, i32, P_i32], C.c_int),
    "orc_block_hashes": ([P_i32, P_i64, i32, i32, P_u64], C.c_int),
    "orc_lpt": ([P_f64, P_i32, i32, i32, i32, i32, P_i64, P_i64], C.c_int),
    "orc_prefix_tables": ([P_i32, P_i64, i32, P_i64, P_i64, P_i64, P_i64, P_i64, P_i64], C.c_int),
    "orc_sweep_select": ([P_f64, P_f64, i64, i32, i32, f64, P_i32], C.c_int),
}


def bind(lib, sigs, prefix=""):
    for name, (args, res) in sigs.items():
        fn = getattr(lib, prefix + name)
        fn.argtypes = args
        fn.restype = res
    return lib
