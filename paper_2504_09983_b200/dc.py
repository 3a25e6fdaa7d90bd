"""ctypes binding of include/dc.h — argument marshalling only.

Every function here forwards to libdc_b200.so with the same name; there is no
Python compute path and no CPU fallback: if the shared library is missing this
module raises at import.  torch is used only to allocate device / pinned
memory and to hand over streams and events.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdc_b200.so")
if os.environ.get("DC_LIB_AB"):      # A/B experiments: another in-tree build of the same library
    LIB_PATH = os.path.join(os.path.dirname(_HERE), os.environ["DC_LIB_AB"])

if not os.path.exists(LIB_PATH):
    raise ImportError("libdc_b200.so not built: run `python -m paper_2504_09983_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)

DC_OK, DC_EINVAL, DC_EOOM, DC_EINFEASIBLE, DC_ECUDA, DC_ESTATE, DC_EPROFILE, DC_ETIMEOUT = range(8)
STATUS = {0: "DC_OK", 1: "DC_EINVAL", 2: "DC_EOOM", 3: "DC_EINFEASIBLE", 4: "DC_ECUDA",
          5: "DC_ESTATE", 6: "DC_EPROFILE", 7: "DC_ETIMEOUT"}
DC_BF16, DC_FP32 = 0, 1
DC_INIT_WEIGHTS, DC_VIRTUAL_RANKS, DC_DEBUG_POISON, DC_DEFER_STATES = 1, 2, 4, 8
DC_PASS_SHARD, DC_PASS_PREFETCH, DC_PASS_UNSHARD, DC_PASS_OFFLOAD, DC_PASS_HOST_STATES = 1, 2, 4, 8, 16
DC_D2H_START, DC_D2H_SYNC_FREE, DC_H2D_START, DC_H2D_SYNC, DC_WRITEBACK = 0, 1, 2, 3, 4


class DCError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


p_i64, p_i32, p_f32, p_u64, vp = C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_float), \
    C.POINTER(C.c_uint64), C.c_void_p


class LayoutArgs(C.Structure):
    _fields_ = [("world", C.c_int32), ("n_params", C.c_int32), ("numel", p_i64), ("layer_of", p_i32),
                ("max_s0_ops", C.c_int32)]


class Layout(C.Structure):
    _fields_ = [("shard_elems", C.c_int64), ("grad_slot_bytes", C.c_int64), ("flag_bytes", C.c_int64),
                ("n_layers", C.c_int32)]


class InitArgs(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32), ("n_params", C.c_int32),
                ("numel", p_i64), ("layer_of", p_i32), ("init_k", p_f32), ("max_s0_ops", C.c_int32),
                ("shard_param", vp), ("master", vp), ("exp_avg", vp), ("exp_avg_sq", vp),
                ("grad_peer_ptrs", p_u64), ("grad_bytes", C.c_uint64),
                ("flag_peer_ptrs", p_u64), ("flag_bytes", C.c_uint64),
                ("host_pinned", vp), ("host_pinned_bytes", C.c_uint64),
                ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("seed", C.c_uint64), ("flags", C.c_uint32), ("spin_limit", C.c_uint32),
                ("micro_steps", C.c_int32), ("grad_acc", vp)]


class PlanOpts(C.Structure):
    _fields_ = [("M_prefetch", C.c_uint64), ("alpha_num", C.c_uint32), ("alpha_den", C.c_uint32),
                ("passes", C.c_uint32), ("strict", C.c_uint32)]


class Fragment(C.Structure):
    _fields_ = [("layer", C.c_int32), ("state", C.c_int32), ("offset_elems", C.c_int64), ("elems", C.c_int64)]


class ModelDims(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("ffn", C.c_int32), ("n_heads", C.c_int32), ("n_kv", C.c_int32),
                ("head_dim", C.c_int32), ("layers", C.c_int32), ("tokens", C.c_int32),
                ("checkpoint", C.c_int32), ("n_experts", C.c_int32)]


class GemmArgs(C.Structure):
    _fields_ = [("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32),
                ("A", vp), ("lda", C.c_int64), ("a_mn_major", C.c_int32),
                ("n_bseg", C.c_int32), ("B", vp * 4), ("ldb", C.c_int64 * 4), ("bseg_end", C.c_int32 * 4),
                ("b_mn_major", C.c_int32), ("b_split_k", C.c_int32),
                ("C", vp), ("ldc", C.c_int64), ("R", vp), ("ldr", C.c_int64), ("num_sms", C.c_int32),
                ("kernel", C.c_int32), ("stream_k", C.c_int32),
                ("epilogue", C.c_int32), ("aux", vp), ("ld_aux", C.c_int64), ("glu_off", C.c_int64),
                ("workspace", vp), ("workspace_bytes", C.c_uint64), ("tile_group_m", C.c_int32),
                ("chunk_flags", vp * 4), ("chunk_S", C.c_int64 * 4), ("chunk_E", C.c_int64 * 4),
                ("chunk_numel", C.c_int64 * 4), ("chunk_value", C.c_uint32 * 4),
                ("chunk_err", vp), ("chunk_timeout_ns", C.c_uint64)]


ctx_p, sched_p, model_p = vp, vp, vp
_sig = {
    "dc_last_error": (C.c_char_p, [vp]),
    "dc_version": (C.c_char_p, []),
    "dc_layout_query": (C.c_int, [C.POINTER(LayoutArgs), C.POINTER(Layout)]),
    "dc_init": (C.c_int, [C.POINTER(InitArgs), C.POINTER(vp)]),
    "dc_destroy": (C.c_int, [vp]),
    "dc_poll": (C.c_int, [vp]),
    "dc_shard_range": (C.c_int, [vp, C.c_int32, p_i64, p_i64]),
    "dc_grad_offset": (C.c_int, [vp, C.c_int32, p_i64]),
    "dc_plan": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(PlanOpts), C.POINTER(vp)]),
    "dc_schedule_json": (C.c_int, [vp, C.c_char_p, C.POINTER(C.c_size_t)]),
    "dc_schedule_capacity": (C.c_uint64, [vp]),
    "dc_schedule_free": (None, [vp]),
    "dc_bind_schedule": (C.c_int, [vp, vp, p_u64, C.c_uint64, vp]),
    "dc_step_begin": (C.c_int, [vp, C.c_int32, vp]),
    "dc_gather_timing": (C.c_int, [vp, vp, vp]),
    "dc_gather": (C.c_int, [vp, C.c_int32, vp, vp]),
    "dc_tensor_ptr": (C.c_int, [vp, C.c_int32, C.POINTER(vp)]),
    "dc_release": (C.c_int, [vp, C.c_int32, vp]),
    "dc_grad_slot": (C.c_int, [vp, C.c_int32, C.POINTER(vp)]),
    "dc_grad_slot_acquire": (C.c_int, [vp, C.c_int32, vp]),
    "dc_grad_slot_publish": (C.c_int, [vp, C.c_int32, vp]),
    "dc_reduce_scatter_step": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_int32, vp]),
    "dc_offload_fragments": (C.c_int, [vp, C.c_int64, C.POINTER(Fragment), p_i32]),
    "dc_offload": (C.c_int, [vp, C.c_int32, C.c_int32, vp]),
    "dc_gemm": (C.c_int, [C.POINTER(GemmArgs), vp]),
    "dc_gemm_pair_slots": (C.c_int32, []),
    "dc_gemm_workspace_bytes": (C.c_uint64, []),
    "dc_model_create": (C.c_int, [vp, C.POINTER(ModelDims), C.POINTER(vp)]),
    "dc_model_destroy": (C.c_int, [vp]),
    "dc_model_act_bytes": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
    "dc_model_bind": (C.c_int, [vp, vp, C.c_uint64, vp, vp]),
    "dc_model_profile_json": (C.c_int, [vp, C.c_char_p, C.POINTER(C.c_size_t)]),
    "dc_model_step": (C.c_int, [vp, C.c_int32, C.c_int32, vp, vp, vp, vp]),
    "dc_model_loss_ptr": (C.c_int, [vp, C.POINTER(p_f32)]),
    "dc_model_act_ptr": (C.c_int, [vp, C.c_int32, C.c_int32, C.POINTER(vp)]),
    "dc_model_launch_count": (C.c_int, [vp, p_i64]),
    "dc_model_set_option": (C.c_int, [vp, C.c_char_p, C.c_int64]),
    "dc_set_option": (C.c_int, [vp, C.c_char_p, C.c_int64]),
    "dc_bind_multicast": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64]),
    "dc_model_join_states": (C.c_int, [vp, vp]),
    "dc_model_graph_capture": (C.c_int, [vp, C.c_int32, vp, vp, vp, vp]),
    "dc_model_graph_launch": (C.c_int, [vp, C.c_int32, vp]),
    "dc_model_host_states_query": (C.c_int, [vp, p_i64, p_i64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "dc_model_bind_host_states": (C.c_int, [vp, vp, vp, vp, C.c_uint64, vp, C.c_uint64]),
}
EXPORTS = tuple(_sig)
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def last_error(ctx=None) -> str:
    s = lib.dc_last_error(ctx)
    return s.decode() if s else ""


def check(status, ctx=None):
    if status != DC_OK:
        raise DCError(status, last_error(ctx))


def call(name, *args, ctx=None):
    check(getattr(lib, name)(*args), ctx)


def _json_out(fn, obj):
    n = C.c_size_t(0)
    check(fn(obj, None, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    n2 = C.c_size_t(n.value + 1)
    check(fn(obj, buf, C.byref(n2)))
    return buf.value.decode()


def schedule_json(sched) -> str:
    return _json_out(lib.dc_schedule_json, sched)


def model_profile_json(model) -> str:
    return _json_out(lib.dc_model_profile_json, model)


def plan(profile_json: str, M: int, M_prefetch=2 << 30, alpha=(3, 2),
         passes=DC_PASS_SHARD | DC_PASS_PREFETCH | DC_PASS_UNSHARD, strict=False):
    """dc_plan -> opaque schedule handle (free with lib.dc_schedule_free)."""
    o = PlanOpts(M_prefetch, alpha[0], alpha[1], passes, 1 if strict else 0)
    out = vp()
    check(lib.dc_plan(profile_json.encode(), M, C.byref(o), C.byref(out)))
    return out


def i64_array(xs):
    return (C.c_int64 * len(xs))(*xs)


def i32_array(xs):
    return (C.c_int32 * len(xs))(*xs)


def f32_array(xs):
    return (C.c_float * len(xs))(*xs)


def u64_array(xs):
    return (C.c_uint64 * len(xs))(*xs)
