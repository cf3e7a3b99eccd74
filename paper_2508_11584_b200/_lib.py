"""ctypes binding of libvpe.so (the C ABI declared in include/vpe.h).

There is no fallback: if the library is missing or fails to load, importing the product path
raises. Build it with ``python -m paper_2508_11584_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

# VPE_LIB selects a diagnostics build (e.g. libvpe_trace.so from VPE_BUILD_TAG=trace) in-tree
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("VPE_LIB", "libvpe.so"))

MAX_LAYERS = 40
MAX_CONSUMERS = 16
HOST_PINNED = -1
DTYPE_CODES = {"f32": 0, "f16_raw": 1, "u8": 2, "i32": 3, "i64": 4, "bf16": 5}

vp = C.c_void_p
i32 = C.c_int32
u32 = C.c_uint32
i64 = C.c_int64
u64 = C.c_uint64
f32 = C.c_float
fptr = C.POINTER(C.c_float)


class TensorSpecC(C.Structure):
    _fields_ = [("label", C.c_char * 64), ("dtype", i32), ("rank", i32), ("dims", i64 * 4)]


class LeaseC(C.Structure):
    _fields_ = [("slot", i32), ("consumer_id", u32), ("frame_id", u64), ("capture_ts", u64), ("consumed", i32)]


class CountersC(C.Structure):
    _fields_ = [("pushed", u64), ("producer_drops", u64), ("evictions", u64), ("consumed", u64), ("resident", u64)]


class VitConfigC(C.Structure):
    _fields_ = [("dim", i32), ("depth", i32), ("heads", i32), ("mlp_hidden", i32), ("resolution", i32),
                ("batch", i32), ("ln_eps", f32), ("taps", i32 * 4)]


L = MAX_LAYERS


class VitWeightsC(C.Structure):
    _fields_ = [("patch_w", vp), ("patch_b", vp), ("cls_pos0", vp), ("pos", vp), ("norm_w", vp), ("norm_b", vp),
                ("ln1_w", vp * L), ("ln1_b", vp * L), ("qkv_w", vp * L), ("qkv_b", vp * L), ("proj_w", vp * L),
                ("proj_b", vp * L), ("ls1", vp * L), ("ln2_w", vp * L), ("ln2_b", vp * L), ("fc1_w", vp * L),
                ("fc1_b", vp * L), ("fc2_w", vp * L), ("fc2_b", vp * L), ("ls2", vp * L)]


class DptConfigC(C.Structure):
    _fields_ = [("dim", i32), ("resolution", i32), ("batch", i32), ("neck", i32 * 4), ("fusion", i32),
                ("head_hidden", i32), ("max_depth", f32)]


class DptWeightsC(C.Structure):
    _fields_ = [("rs_w", vp * 4), ("rs_b", vp * 4), ("rs3_conv_w", vp), ("rs3_conv_b", vp), ("neck_w", vp * 4),
                ("proj_w", vp * 4), ("proj_b", vp * 4), ("rcu_w", (vp * 4) * 4), ("rcu_b", (vp * 4) * 4),
                ("head1_w", vp), ("head1_b", vp), ("head2_w", vp), ("head2_b", vp), ("head3_w", vp),
                ("head3_b", f32)]


class SegConfigC(C.Structure):
    _fields_ = [("dim", i32), ("resolution", i32), ("batch", i32), ("classes", i32)]


class SegWeightsC(C.Structure):
    _fields_ = [("w_split", vp), ("b", vp)]


class DetConfigC(C.Structure):
    _fields_ = [("dim", i32), ("resolution", i32), ("batch", i32), ("pre_nms_top_n", i32), ("post_nms_top_n", i32),
                ("nms_thresh", f32), ("min_size", f32), ("score_thresh", f32), ("num_anchors", i32),
                ("base_anchors", (f32 * 4) * 9), ("bbox_clip", f32)]


class DetWeightsC(C.Structure):
    _fields_ = [("conv_w_split", vp), ("conv_b", vp), ("cls_w", vp), ("cls_b", vp), ("box_w", vp), ("box_b", vp)]


class DetOutputsC(C.Structure):
    _fields_ = [("boxes", vp), ("scores", vp), ("index", vp), ("count", vp), ("objectness", vp), ("deltas", vp),
                ("top_index", vp)]


_SIGS = {
    # atomics
    "vpe_atomic_check_base": (i32, [vp, C.c_size_t]),
    "vpe_u32_load": (i32, [vp, C.c_size_t, i64, C.POINTER(u32)]),
    "vpe_u32_store": (i32, [vp, C.c_size_t, i64, u32]),
    "vpe_u32_cas": (i32, [vp, C.c_size_t, i64, u32, u32, C.POINTER(u32)]),
    "vpe_u64_load": (i32, [vp, C.c_size_t, i64, C.POINTER(u64)]),
    "vpe_u64_store": (i32, [vp, C.c_size_t, i64, u64]),
    "vpe_u64_add": (i32, [vp, C.c_size_t, i64, u64, C.POINTER(u64)]),
    "vpe_busy_spin_ns": (None, [i64]),
    "vpe_now_ns": (i64, []),
    # ring
    "vpe_ring_create": (i32, [C.POINTER(TensorSpecC), i32, i32, i32, i32, C.POINTER(vp)]),
    "vpe_ring_destroy": (i32, [vp]),
    "vpe_ring_create_shared": (i32, [C.POINTER(TensorSpecC), i32, i32, i32, i32, C.c_char_p, C.POINTER(vp)]),
    "vpe_ring_attach": (i32, [C.c_char_p, C.POINTER(vp)]),
    "vpe_ring_header": (i32, [vp, C.POINTER(vp), C.POINTER(C.c_size_t)]),
    "vpe_ring_data": (i32, [vp, C.POINTER(vp), C.POINTER(C.c_size_t)]),
    "vpe_ring_slot_ptr": (i32, [vp, i32, i32, C.POINTER(vp)]),
    "vpe_ring_label_offset": (i32, [vp, i32, i32, C.POINTER(i64)]),
    "vpe_ring_claim": (i32, [vp, u64, u64, vp, C.POINTER(i32), C.POINTER(u64), C.POINTER(i32)]),
    "vpe_ring_publish": (i32, [vp, i32, vp]),
    "vpe_ring_abort": (i32, [vp, i32]),
    "vpe_ring_register_consumer": (i32, [vp, u32, C.POINTER(i32)]),
    "vpe_ring_last_consumed": (i32, [vp, u32, C.POINTER(u64)]),
    "vpe_ring_acquire_latest": (i32, [vp, u32, vp, C.POINTER(LeaseC)]),
    "vpe_ring_commit": (i32, [vp, C.POINTER(LeaseC), vp]),
    "vpe_ring_consume": (i32, [vp, C.POINTER(LeaseC), C.POINTER(i32), i32, C.POINTER(vp), vp]),
    "vpe_ring_release": (i32, [vp, C.POINTER(LeaseC), vp]),
    "vpe_ring_pop": (i32, [vp, u32, C.POINTER(vp), i32, vp, C.POINTER(LeaseC)]),
    "vpe_ring_counters": (i32, [vp, C.POINTER(CountersC)]),
    "vpe_ring_slot_state": (i32, [vp, i32, C.POINTER(u32), C.POINTER(u64)]),
    "vpe_copy_counter": (i64, []),
    "vpe_region_create": (i32, [C.c_char_p, u64, i32, C.POINTER(vp)]),
    "vpe_region_attach": (i32, [C.c_char_p, u64, C.POINTER(vp)]),
    "vpe_region_info": (i32, [vp, C.POINTER(vp), C.POINTER(u64), C.POINTER(i32)]),
    "vpe_region_destroy": (i32, [vp, i32]),
    "vpe_copy_out": (i32, [vp, vp, u64, vp, i32]),
    # models
    "vpe_vit_create": (i32, [C.POINTER(VitConfigC), C.POINTER(VitWeightsC), C.POINTER(vp)]),
    "vpe_vit_destroy": (i32, [vp]),
    "vpe_vit_forward": (i32, [vp, vp, C.POINTER(vp), vp]),
    "vpe_vit_residual": (i32, [vp, C.POINTER(vp)]),
    "vpe_vit_forward_camera": (i32, [vp, vp, i32, i32, C.POINTER(vp), vp]),
    "vpe_op_camera_im2col": (i32, [vp, i32, i32, i32, i32, vp, vp]),
    "vpe_dpt_create": (i32, [C.POINTER(DptConfigC), C.POINTER(DptWeightsC), C.POINTER(vp)]),
    "vpe_dpt_destroy": (i32, [vp]),
    "vpe_dpt_forward": (i32, [vp, C.POINTER(vp), vp, vp, vp]),
    "vpe_seg_create": (i32, [C.POINTER(SegConfigC), C.POINTER(SegWeightsC), C.POINTER(vp)]),
    "vpe_seg_destroy": (i32, [vp]),
    "vpe_seg_forward": (i32, [vp, vp, vp, vp, vp]),
    "vpe_det_create": (i32, [C.POINTER(DetConfigC), C.POINTER(DetWeightsC), C.POINTER(vp)]),
    "vpe_det_destroy": (i32, [vp]),
    "vpe_det_forward": (i32, [vp, vp, C.POINTER(DetOutputsC), vp]),
    # ops
    "vpe_op_linear": (i32, [vp, i32, i32, vp, i32, i32, vp, vp, vp, i32, i32, i32, vp]),
    "vpe_op_conv": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, i32, vp, vp, vp, vp, vp, i32, i32, vp]),
    "vpe_set_pdl": (i32, [i32]),
    "vpe_set_dpt_branches": (i32, [i32]),
    "vpe_debug_att_trace": (i32, [vp, i32]),
    "vpe_debug_gemm_trace": (i32, [vp, i32]),
    "vpe_op_attention": (i32, [vp, vp, i32, i32, i32, i32, vp]),
    "vpe_op_linear_resid_ln": (i32, [vp, i32, i32, vp, vp, vp, vp, vp, vp, f32, vp, vp, vp, vp, vp]),
    "vpe_op_conv_up_pack": (i32, [vp, i32, vp, vp]),
    "vpe_op_conv_up": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, i32, vp, vp, i32, i32, vp, f32, vp, vp]),
    "vpe_op_bilinear": (i32, [vp, i32, i32, i32, i32, i32, vp, i32, i32, vp]),
    "vpe_op_upsample_argmax": (i32, [vp, i32, i32, i32, i32, i32, vp, vp]),
    "vpe_op_layernorm": (i32, [vp, i32, i32, vp, vp, f32, vp, vp, vp, vp, vp]),
    # runtime
    "vpe_stream_create": (i32, [i32, C.POINTER(vp)]),
    "vpe_stream_destroy": (i32, [vp]),
    "vpe_stream_sync": (i32, [vp]),
    "vpe_graph_begin": (i32, [vp]),
    "vpe_graph_end": (i32, [vp, C.POINTER(vp)]),
    "vpe_graph_launch": (i32, [vp, vp]),
    "vpe_graph_destroy": (i32, [vp]),
    "vpe_event_create": (i32, [C.POINTER(vp)]),
    "vpe_event_record": (i32, [vp, vp]),
    "vpe_event_sync": (i32, [vp]),
    "vpe_event_elapsed_ms": (i32, [vp, vp, C.POINTER(f32)]),
    "vpe_event_destroy": (i32, [vp]),
    "vpe_stream_wait_event": (i32, [vp, vp]),
    "vpe_memcpy_async": (i32, [vp, vp, C.c_size_t, vp]),
    "vpe_kernel_launches": (i64, []),
    "vpe_status_str": (C.c_char_p, [i32]),
}

EXPORTS = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libvpe.so not built at {LIB_PATH}; run `python -m paper_2508_11584_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int, what: str = "") -> int:
    """Raise the reference's exception class for an error status; pass OK and outcomes."""
    if rc in (errors.OK, errors.OVERFLOW_REJECTED, errors.NO_NEW_DATA):
        return rc
    exc = errors.STATUS.get(rc, errors.EngineError)
    msg = lib.vpe_status_str(rc).decode()
    raise exc(f"{what}: {msg} (status {rc})" if what else f"{msg} (status {rc})")


def ptr(t) -> int:
    """Raw data pointer of a torch tensor (or None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()
