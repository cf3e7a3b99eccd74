/*
 * vpe.h — C ABI of libvpe.so, the B200-native (sm_100a) hot path of VPEngine
 * (arXiv 2508.11584): a shared DINOv2 backbone that writes its tap features once into a
 * device-resident ring, consumed in place by depth / segmentation / detection heads.
 *
 * Plain pointers and sizes only (no torch types). Every entry point returns an int status
 * that maps 1:1 onto the reference's exception classes (fanpipe/errors.py:4-53), plus the
 * two non-error outcomes of the channel API (PushKind.OVERFLOW_REJECTED, "no new data").
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/fanpipe/):
 *   vpe_u32_* / vpe_u64_* / vpe_busy_spin_ns  <- _kernels.pyx:56-109  (AtomicBuffer, busy_spin_ns)
 *   vpe_ring_create / _destroy                <- channels.py:537-576    (create_channel)
 *   vpe_ring_header / _data / _slot_ptr       <- channels.py:14-26, 232-247 (header + group views)
 *   vpe_ring_claim + vpe_ring_publish/_abort  <- channels.py:274-331    (Channel.push / _claim_slot)
 *   vpe_ring_register_consumer                <- channels.py:335-358
 *   vpe_ring_acquire_latest                   <- channels.py:423-452
 *   vpe_ring_consume                          <- channels.py:454-474    (copy_out per label)
 *   vpe_ring_commit  (new: in-place consume)  <- channels.py:470-473    (cursor advance, no copy)
 *   vpe_ring_release                          <- channels.py:476-489
 *   vpe_ring_pop                              <- channels.py:377-421
 *   vpe_ring_counters                         <- channels.py:493-504
 *   vpe_copy_counter                          <- arena.py:190-219
 *   vpe_region_* / vpe_copy_out               <- arena.py:285-373    (create/attach_region, copy_out)
 *   vpe_vit_* / vpe_dpt_* / vpe_seg_* / vpe_det_* <- SPEC.md:232-243 ComputeBackend.infer
 *        (the reference has no NN code; these are the backend descriptors "b200_vit",
 *         "b200_dpt", "b200_linseg", "b200_det" that stand in for TensorRT engines)
 */
#ifndef VPE_H
#define VPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-53) ---- */
enum {
  VPE_OK = 0,
  VPE_E_ENGINE = 1,          /* EngineError */
  VPE_E_ALREADY_EXISTS = 2,  /* AlreadyExists */
  VPE_E_NOT_FOUND = 3,       /* NotFound */
  VPE_E_RESOURCE = 4,        /* ResourceError */
  VPE_E_CORRUPT_HANDLE = 5,  /* CorruptHandle */
  VPE_E_SHAPE = 6,           /* ShapeError */
  VPE_E_LABEL = 7,           /* LabelError */
  VPE_E_USE_AFTER_CONSUME = 8, /* UseAfterConsume */
  VPE_E_WRITER = 9,          /* WriterError */
  VPE_E_CONFIG = 10,         /* ConfigError */
  VPE_E_PROTOCOL = 11,       /* ProtocolError */
  VPE_E_STARTUP = 12,        /* StartupError */
  VPE_E_CORRUPT_CARD = 13,   /* CorruptCard */
  VPE_E_VALUE = 20,          /* ValueError (bad atomic offset, frame-id order) */
  VPE_E_RUNTIME = 21,        /* RuntimeError (release of an unleased slot) */
  VPE_E_CUDA = 30,           /* CUDA runtime / driver failure */
  VPE_OVERFLOW_REJECTED = 100, /* PushKind.OVERFLOW_REJECTED (not an error) */
  VPE_NO_NEW_DATA = 101        /* acquire_latest -> None, pop -> None */
};

/* ---- dtypes (arena.py:42-65, plus additive BF16) ---- */
enum { VPE_F32 = 0, VPE_F16_RAW = 1, VPE_U8 = 2, VPE_I32 = 3, VPE_I64 = 4, VPE_BF16 = 5 };
enum { VPE_FIFO = 0, VPE_LATEST = 1 };               /* ChannelMode, channels.py:68-70 */
#define VPE_MAX_CONSUMERS 16                         /* channels.py:58 */
#define VPE_HOST_PINNED (-1)                         /* ring data in pinned host memory */
#define VPE_HOST_PLAIN (-2)                          /* ring data in pageable host memory, no CUDA (tests) */

/* ---- atomics over a caller-owned buffer (replaces fanpipe._kernels.AtomicBuffer) ---- */
int vpe_atomic_check_base(const void* base, size_t size);
int vpe_u32_load(void* base, size_t size, int64_t off, uint32_t* out);
int vpe_u32_store(void* base, size_t size, int64_t off, uint32_t value);
int vpe_u32_cas(void* base, size_t size, int64_t off, uint32_t expected, uint32_t desired, uint32_t* prev);
int vpe_u64_load(void* base, size_t size, int64_t off, uint64_t* out);
int vpe_u64_store(void* base, size_t size, int64_t off, uint64_t value);
int vpe_u64_add(void* base, size_t size, int64_t off, uint64_t delta, uint64_t* prev);
void vpe_busy_spin_ns(int64_t duration_ns);
int64_t vpe_now_ns(void);

/* ---- device feature ring (LATEST) / output queue (FIFO) ---- */
typedef struct vpe_ring vpe_ring;
typedef struct {
  char label[64];
  int32_t dtype;
  int32_t rank;
  int64_t dims[4];
} vpe_tensor_spec;
typedef struct {
  int32_t slot;
  uint32_t consumer_id;
  uint64_t frame_id;
  uint64_t capture_ts;
  int32_t consumed;
} vpe_lease;
typedef struct {
  uint64_t pushed, producer_drops, evictions, consumed, resident;
} vpe_counters;

int vpe_ring_create(const vpe_tensor_spec* specs, int32_t nspecs, int32_t capacity, int32_t mode, int32_t device,
                    vpe_ring** out);
int vpe_ring_destroy(vpe_ring* r);
/* Cross-process rings (channels.py:537-594 create_channel / open_channel across processes):
 * the control block goes to POSIX shm "/vpe.<name>-c", the HBM arena and the ready/done events
 * are exported through CUDA IPC (handles in "/vpe.<name>-x"); a VPE_HOST_PLAIN ring keeps its
 * data in "/vpe.<name>-d". The creator unlinks the segments on destroy. */
int vpe_ring_create_shared(const vpe_tensor_spec* specs, int32_t nspecs, int32_t capacity, int32_t mode,
                           int32_t device, const char* name, vpe_ring** out);
int vpe_ring_attach(const char* name, vpe_ring** out);
int vpe_ring_header(vpe_ring* r, void** base, size_t* size);
int vpe_ring_data(vpe_ring* r, void** base, size_t* size);
int vpe_ring_slot_ptr(vpe_ring* r, int32_t slot, int32_t label, void** ptr);
int vpe_ring_label_offset(vpe_ring* r, int32_t slot, int32_t label, int64_t* offset);
/* producer: FREE slot, else (LATEST) the oldest READY slot with no leases; the producer stream
 * waits on every consumer's last "done" event for the slot (WAR hazard). */
int vpe_ring_claim(vpe_ring* r, uint64_t frame_id, uint64_t capture_ts, void* stream, int32_t* slot,
                   uint64_t* evicted_frame_id, int32_t* evicted);
int vpe_ring_publish(vpe_ring* r, int32_t slot, void* stream); /* records ready event, state READY */
int vpe_ring_abort(vpe_ring* r, int32_t slot);                  /* writer failed -> FREE */
int vpe_ring_register_consumer(vpe_ring* r, uint32_t consumer_id, int32_t* capacity_warning);
int vpe_ring_last_consumed(vpe_ring* r, uint32_t consumer_id, uint64_t* frame_id);
/* lease the newest READY frame newer than the consumer cursor; the consumer stream waits on
 * the slot's ready event. VPE_NO_NEW_DATA when nothing newer exists. */
int vpe_ring_acquire_latest(vpe_ring* r, uint32_t consumer_id, void* stream, vpe_lease* lease);
/* in-place consumption done: records the consumer's done event on `stream`, advances the
 * cursor, drops the lease (no copy). */
int vpe_ring_commit(vpe_ring* r, vpe_lease* lease, void* stream);
/* copy the selected labels (async D2D/D2H on `stream`, copy counter +1 per label), then commit */
int vpe_ring_consume(vpe_ring* r, vpe_lease* lease, const int32_t* labels, int32_t nlabels, void* const* dst,
                     void* stream);
int vpe_ring_release(vpe_ring* r, vpe_lease* lease, void* stream);
/* FIFO: oldest READY frame copied into dst (all labels), slot FREE after copy. dst_on_host != 0:
 * dst are host pointers, the call waits for the producer's ready event and copies synchronously;
 * otherwise dst are device pointers and the copies are ordered on `stream` (NULL = the legacy
 * default stream). Streams are never NULL-tested: NULL is a valid stream for every entry point. */
int vpe_ring_pop(vpe_ring* r, uint32_t consumer_id, void* const* dst, int32_t dst_on_host, void* stream,
                 vpe_lease* envelope);
int vpe_ring_counters(vpe_ring* r, vpe_counters* c);
int vpe_ring_slot_state(vpe_ring* r, int32_t slot, uint32_t* state, uint64_t* frame_id);
int64_t vpe_copy_counter(void);

/* ---- shareable regions (arena.py:285-413 create_region / attach_region / copy_out) ----
 * name = "<namespace>.<region>"; a POSIX segment "/<name>" holds the bytes (VPE_HOST_PLAIN) or a
 * descriptor of the HBM allocation exported through CUDA IPC (device >= 0). Zero-initialised.
 * Errors: AlreadyExists / NotFound / CorruptHandle (attach with expect_bytes > region size). */
typedef struct vpe_region vpe_region;
int vpe_region_create(const char* name, uint64_t nbytes, int32_t device, vpe_region** out);
int vpe_region_attach(const char* name, uint64_t expect_bytes, vpe_region** out);
int vpe_region_info(vpe_region* region, void** base, uint64_t* nbytes, int32_t* device);
int vpe_region_destroy(vpe_region* region, int32_t unlink_segment);
/* the single permitted copy (copy counter +1): host memcpy, or stream-ordered cudaMemcpyAsync
 * when either side is device memory (host_sync != 0: wait for it) */
int vpe_copy_out(void* dst, const void* src, uint64_t nbytes, void* stream, int32_t host_sync);

/* ---- backbone: DINOv2 ViT forward writing 4 tap features (bf16 [B,T,D]) ---- */
#define VPE_MAX_LAYERS 40
typedef struct {
  int32_t dim, depth, heads, mlp_hidden, resolution, batch;
  float ln_eps;
  int32_t taps[4]; /* 1-based block indices, ascending; taps[3] == depth */
} vpe_vit_config;
typedef struct {
  const void* patch_w;   /* bf16 [D, 640]: conv weight flattened (c,ky,kx), K zero-padded 588->640 */
  const float* patch_b;  /* [D] */
  const float* cls_pos0; /* [D] cls_token + pos[0] */
  const float* pos;      /* [T, D] position embedding interpolated to the grid */
  const float* norm_w;   /* final LayerNorm (applied at every tap) */
  const float* norm_b;
  const float* ln1_w[VPE_MAX_LAYERS];
  const float* ln1_b[VPE_MAX_LAYERS];
  const void* qkv_w[VPE_MAX_LAYERS];  /* bf16 [3D, D] (query | key | value rows) */
  const float* qkv_b[VPE_MAX_LAYERS]; /* [3D] */
  const void* proj_w[VPE_MAX_LAYERS]; /* bf16 [D, D] */
  const float* proj_b[VPE_MAX_LAYERS];
  const float* ls1[VPE_MAX_LAYERS];
  const float* ln2_w[VPE_MAX_LAYERS];
  const float* ln2_b[VPE_MAX_LAYERS];
  const void* fc1_w[VPE_MAX_LAYERS]; /* bf16 [4D, D] */
  const float* fc1_b[VPE_MAX_LAYERS];
  const void* fc2_w[VPE_MAX_LAYERS]; /* bf16 [D, 4D] */
  const float* fc2_b[VPE_MAX_LAYERS];
  const float* ls2[VPE_MAX_LAYERS];
} vpe_vit_weights;
typedef struct vpe_vit vpe_vit;
int vpe_vit_create(const vpe_vit_config* cfg, const vpe_vit_weights* w, vpe_vit** out);
int vpe_vit_destroy(vpe_vit* v);
/* pixels: u8 [B,3,R,R] device; taps: 4 device pointers to bf16 [B,T,D] (ring slot labels) */
int vpe_vit_forward(vpe_vit* v, const void* pixels_u8, void* const* taps, void* stream);
/* Camera ingest fused into the patch embedding: frames_hwc_u8 is [batch, height,
 * width, 3] u8 (any size): centre-cropped to a square, bilinearly resized to resolution
 * (align_corners=False, no antialias), ImageNet-normalised, then the same forward. */
int vpe_vit_forward_camera(vpe_vit* v, const void* frames_hwc_u8, int32_t height, int32_t width,
                           void* const* taps, void* stream);
/* debug: fp32 residual stream [B*T, D] after the last forward */
int vpe_vit_residual(vpe_vit* v, const float** resid);

/* ---- DPT depth head ---- */
typedef struct {
  int32_t dim, resolution, batch;
  int32_t neck[4];
  int32_t fusion, head_hidden;
  float max_depth;
} vpe_dpt_config;
typedef struct {
  /* reassemble: [0],[1] = 1x1 proj composed with ConvT (bf16 [k*k*C_i, D], bias fp32 [k*k*C_i]);
   * [2] = 1x1 proj (bf16 [C_2, D]); [3] = 1x1 proj (bf16 [D', D]) then 3x3 s2 conv (bf16 [C_3, 9*D']) */
  const void* rs_w[4];
  const float* rs_b[4];
  const void* rs3_conv_w;  /* bf16 [C3, 9*C3] (tap-major, channel) */
  const float* rs3_conv_b;
  const void* neck_w[4];   /* bf16 [F, 9*Cpad_i], no bias */
  const void* proj_w[4];   /* fusion projection bf16 [F, F] */
  const float* proj_b[4];
  const void* rcu_w[4][4]; /* [layer][rcu1.conv1, rcu1.conv2, rcu2.conv1, rcu2.conv2] bf16 [F, 9F] */
  const float* rcu_b[4][4];
  const void* head1_w;     /* bf16 [F/2, 9F] */
  const float* head1_b;
  const void* head2_w;     /* bf16 [Hh, 9*F/2] */
  const float* head2_b;
  const float* head3_w;    /* [Hh] */
  float head3_b;
} vpe_dpt_weights;
typedef struct vpe_dpt vpe_dpt;
int vpe_dpt_create(const vpe_dpt_config* cfg, const vpe_dpt_weights* w, vpe_dpt** out);
int vpe_dpt_destroy(vpe_dpt* d);
/* taps: 4 x bf16 [B,T,D]; depth: f32 [B,R,R]; depth_pre (nullable): pre-final-ReLU map */
int vpe_dpt_forward(vpe_dpt* d, const void* const* taps, float* depth, float* depth_pre, void* stream);

/* ---- linear segmentation head ---- */
typedef struct {
  int32_t dim, resolution, batch, classes;
} vpe_seg_config;
typedef struct {
  const void* w_split; /* bf16 [Cpad, 2D]: BN-folded classifier, hi | lo split */
  const float* b;      /* [C] BN-folded bias */
} vpe_seg_weights;
typedef struct vpe_seg vpe_seg;
int vpe_seg_create(const vpe_seg_config* cfg, const vpe_seg_weights* w, vpe_seg** out);
int vpe_seg_destroy(vpe_seg* s);
/* final: bf16 [B,T,D]; labels: u8 [B,R,R]; logits (nullable): f32 [B, h*h, C] */
int vpe_seg_forward(vpe_seg* s, const void* final_tap, uint8_t* labels, float* logits, void* stream);

/* ---- RPN-style detection head ---- */
typedef struct {
  int32_t dim, resolution, batch;
  int32_t pre_nms_top_n, post_nms_top_n;
  float nms_thresh, min_size, score_thresh;
  int32_t num_anchors;
  float base_anchors[9][4];
  float bbox_clip;
} vpe_det_config;
typedef struct {
  const void* conv_w_split; /* bf16 [D, 2*9*D]: 3x3 conv, hi | lo split, tap-major */
  const float* conv_b;      /* [D] */
  const float* cls_w;       /* f32 [A, D] */
  const float* cls_b;       /* [A] */
  const float* box_w;       /* f32 [4A, D] */
  const float* box_b;       /* [4A] */
} vpe_det_weights;
typedef struct {
  float* boxes;      /* [B, post, 4] */
  float* scores;     /* [B, post] */
  int64_t* index;    /* [B, post] anchor index into the (y, x, a) flattening */
  int32_t* count;    /* [B] */
  float* objectness; /* nullable [B, h*h*A] logits */
  float* deltas;     /* nullable [B, h*h*A, 4] */
  int64_t* top_index;/* nullable [B, pre] pre-NMS top-k (descending logit) */
} vpe_det_outputs;
typedef struct vpe_det vpe_det;
int vpe_det_create(const vpe_det_config* cfg, const vpe_det_weights* w, vpe_det** out);
int vpe_det_destroy(vpe_det* d);
int vpe_det_forward(vpe_det* d, const void* final_tap, const vpe_det_outputs* out, void* stream);

/* ---- single-op entry points (parity tests, microbenchmarks) ---- */
/* out = epilogue(A[M,K] * W[N,K]^T): kind 0 bf16 (+act 0 none/1 gelu/2 relu), 1 resid f32 += scale*(.),
 * 3 f32. Kw may be a multiple of K (split-precision weights, A repeated). */
int vpe_op_linear(const void* A, int32_t M, int32_t K, const void* W, int32_t N, int32_t Kw, const float* bias,
                  const float* scale, void* out, int32_t kind, int32_t act, int32_t bn, void* stream);
/* bn: 128 x bn tiles (32, 64, 128, 192, 256) */
/* resid fp32 [M, 384] += ls * (A W^T + bias), A bf16 [M, K], W bf16 [384, K]; then xln bf16 =
 * LayerNorm(resid) (ln_w, ln_b) and optionally tap_out = LayerNorm(resid) (tap_w, tap_b), in the
 * same kernel (DINOv2 block: attention.output / mlp.fc2 + layer_scale + residual, then the next
 * norm: modeling_dinov2.py:382-420) */
int vpe_op_linear_resid_ln(const void* A, int32_t M, int32_t K, const void* W, const float* bias, const float* ls,
                           float* resid, const float* ln_w, const float* ln_b, float eps, void* xln, const float* tap_w,
                           const float* tap_b, void* tap_out, void* stream);
/* camera ingest alone: [B,H,W,3] u8 -> normalised bf16 patch rows [B*(R/14)^2, 640] (k = c*196+ky*14+kx) */
int vpe_op_camera_im2col(const void* frames_hwc_u8, int32_t B, int32_t height, int32_t width, int32_t resolution,
                         void* out_bf16, void* stream);
/* 3x3 or 1x1 same-padding conv on NHWC bf16 x [B,H,W,Cp] with weights [N, ks*ks*Cp] -> out bf16 NHWC
 * [B,H,W,ldo]; out = act(conv + bias + add1 + add2); out_relu optional */
int vpe_op_conv(const void* x, int32_t B, int32_t H, int32_t W, int32_t C, int32_t Cp, int32_t ks, const void* w,
                int32_t N, const float* bias, const void* add1, const void* add2, void* out, void* out_relu,
                int32_t ldo, int32_t act, void* stream);
/* conv of the resize: 3x3 same-padding conv applied to the bilinear align_corners=True resize of
 * x [B,Hs,Ws,Cp] (Cp = 32 or 64) to Ho x Wo, the resized map never materialised; out bf16 NHWC
 * [B,Ho,Wo,ldo] = act(conv + bias). Bit-identical to vpe_op_bilinear followed by vpe_op_conv (DPT
 * head: modeling_depth_anything.py:288-308). Weights [N = 32, 9*Cp] tap-major, first packed by
 * vpe_op_conv_up_pack into wpack (3*96*Cp bf16). With w3: the DPT depth epilogue instead,
 * depth[B,Ho,Wo] f32 = relu(b3 + sum_c relu(conv_c + bias_c) w3_c) */
int vpe_op_conv_up_pack(const void* w, int32_t Cp, void* wpack, void* stream);
int vpe_op_conv_up(const void* x, int32_t B, int32_t Hs, int32_t Ws, int32_t Cp, int32_t Ho, int32_t Wo,
                   const void* wpack, int32_t N, const float* bias, void* out, int32_t ldo, int32_t act,
                   const float* w3, float b3, float* depth, void* stream);
int vpe_op_attention(const void* qkv, void* out, int32_t B, int32_t T, int32_t D, int32_t heads, void* stream);
/* bilinear (align_corners=False) upsample of fp32 logits [B, h*h, cp] (C real classes) to
 * [B, R, R] + argmax over classes -> u8 labels; R = 14 h; torch's rounding and first-index ties
 * (reference seg head: SPEC.md:232-243, oracle/seg.py seg_forward) */
int vpe_op_upsample_argmax(const float* logits, int32_t B, int32_t h, int32_t C, int32_t cp, int32_t resolution,
                           uint8_t* labels, void* stream);
/* bilinear resize, align_corners=True, NHWC bf16 [B,Hi,Wi,cp] -> [B,Ho,Wo,cp] (first C channels)
 * (DPT fusion/head upsampling: modeling_depth_anything.py:157-200, 288-293) */
int vpe_op_bilinear(const void* in, int32_t B, int32_t Hi, int32_t Wi, int32_t cp, int32_t C, void* out, int32_t Ho,
                    int32_t Wo, void* stream);
int vpe_op_layernorm(const float* x, int32_t M, int32_t D, const float* w, const float* b, float eps, void* out_bf16,
                     const float* w2, const float* b2, void* out2_bf16, void* stream);

/* ---- CUDA graph + stream helpers (one process per GPU, priority streams) ---- */
typedef struct vpe_graph vpe_graph;
int vpe_stream_create(int32_t priority, void** stream); /* lower number = higher priority */
int vpe_stream_destroy(void* stream);
int vpe_stream_sync(void* stream);
int vpe_graph_begin(void* stream);
int vpe_graph_end(void* stream, vpe_graph** out);
int vpe_graph_launch(vpe_graph* g, void* stream);
int vpe_graph_destroy(vpe_graph* g);
int vpe_event_create(void** ev);
int vpe_event_record(void* ev, void* stream);
int vpe_event_sync(void* ev);   /* host waits for the event (GIL released by ctypes) */
int vpe_event_elapsed_ms(void* start, void* end, float* ms);
int vpe_event_destroy(void* ev);
int vpe_stream_wait_event(void* stream, void* ev);
int vpe_memcpy_async(void* dst, const void* src, size_t bytes, void* stream);
int64_t vpe_kernel_launches(void); /* kernels enqueued by libvpe since load (graph replays count per node) */
/* programmatic dependent launch for the backbone kernels enqueued (or graph-captured) from now
 * on: 0 off, 1 dependents released at kernel start, 2 released after each persistent kernel's last
 * TMA load (see csrc/util.cuh); VPE_PDL / VPE_PDL_LATE env override */
int vpe_set_pdl(int32_t on);
/* DPT reassemble / neck branches 0..2 on side streams (forked and joined with events, so
 * graph capture records the DAG) for forwards enqueued from now on: -1 auto (on below batch 8,
 * the default), 0 off, 1 on; VPE_DPT_BRANCHES env sets the initial mode */
int vpe_set_dpt_branches(int32_t mode);
const char* vpe_status_str(int status);
/* diagnostics: timeline of attention CTA 0 when the process runs with VPE_ATT_TRACE=1
   ((code, clock64) pairs; see csrc/attention.cu) */
int vpe_debug_att_trace(unsigned long long* host, int32_t n);
int vpe_debug_gemm_trace(unsigned long long* host, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* VPE_H */
