// Device feature ring: the reference's LATEST/FIFO channel state machine
// (fanpipe/channels.py:1-594) over an HBM (or pinned-host) slot arena, with CUDA-event
// producer/consumer handoff instead of bytes-visible-on-store.
//
// The control block keeps the reference's PECH1 header layout byte for byte
// (channels.py:14-26): magic, mode u8 @6, capacity u32 @8, slot records stride 24 from 16
// {state u32, frame_id u64 @8, capture_ts u64 @16}, 16 cursor entries stride 16
// {consumer_id u32, last_frame u64 @8}, then producer_drops, evictions, pushed, consumed (u64).
// State words use the reference's acquire/release CAS protocol (_kernels.pyx:18-37).
//
// GPU meaning of the states: READY = the producer's writes are *enqueued* and the slot's ready
// event is recorded on the producer stream; every lease makes the consumer stream wait on that
// event (RAW). A consumer's commit records its done event; a producer re-claiming the slot makes
// its stream wait on every consumer's last done event for that slot (WAR). So host-side lease
// counting orders the host, events order the device.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>

#include "util.cuh"

namespace {

constexpr uint32_t STATE_FREE = 0, STATE_WRITING = 1, STATE_READY = 2;
constexpr int SLOT0 = 16, SLOT_STRIDE = 24, CURSOR_STRIDE = 16;
constexpr int ALIGN = 64, ARENA_HDR = 64;
std::atomic<int64_t> g_copies{0};

inline uint32_t ld32(const void* p) { return __atomic_load_n(static_cast<const uint32_t*>(p), __ATOMIC_ACQUIRE); }
inline void st32(void* p, uint32_t v) { __atomic_store_n(static_cast<uint32_t*>(p), v, __ATOMIC_RELEASE); }
inline uint32_t cas32(void* p, uint32_t expected, uint32_t desired) {
  __atomic_compare_exchange_n(static_cast<uint32_t*>(p), &expected, desired, false, __ATOMIC_ACQ_REL,
                              __ATOMIC_ACQUIRE);
  return expected;
}
inline uint64_t ld64(const void* p) { return __atomic_load_n(static_cast<const uint64_t*>(p), __ATOMIC_ACQUIRE); }
inline void st64(void* p, uint64_t v) { __atomic_store_n(static_cast<uint64_t*>(p), v, __ATOMIC_RELEASE); }
inline uint64_t add64(void* p, uint64_t v) { return __atomic_fetch_add(static_cast<uint64_t*>(p), v, __ATOMIC_ACQ_REL); }

int itemsize(int dt) {
  switch (dt) {
    case VPE_F32: return 4;
    case VPE_F16_RAW: return 2;
    case VPE_U8: return 1;
    case VPE_I32: return 4;
    case VPE_I64: return 8;
    case VPE_BF16: return 2;
    default: return 0;
  }
}

size_t align_up(size_t n, size_t a) { return (n + a - 1) / a * a; }

}  // namespace

struct vpe_ring {
  int nspecs = 0, capacity = 0, mode = 0, device = 0;
  vpe_tensor_spec* specs = nullptr;
  size_t* nbytes = nullptr;   // per label
  size_t* offsets = nullptr;  // [capacity * nspecs], data-area relative (ArenaLayout)
  uint8_t* hdr = nullptr;
  size_t hdr_bytes = 0;
  uint8_t* data = nullptr;  // region base (64-byte PEAR1 header, then the data area)
  size_t data_bytes = 0;
  cudaEvent_t* ready = nullptr;       // [capacity]
  cudaEvent_t* done = nullptr;        // [capacity * MAX_CONSUMERS]
  uint8_t* done_valid = nullptr;      // [capacity * MAX_CONSUMERS] (in the IPC segment when shared)
  // cross-process sharing: 0 private, 1 creator of the shm segments, 2 attached
  int role = 0;
  char nm_hdr[192] = {0}, nm_ipc[192] = {0}, nm_dat[192] = {0};
  uint8_t* ipc = nullptr;
  size_t ipc_bytes = 0;
  int64_t* pending_evict = nullptr;   // [capacity], -1 none
  uint64_t last_id = 0, last_ts = 0;
  int cursor_slot[VPE_MAX_CONSUMERS];
  uint32_t cursor_ids[VPE_MAX_CONSUMERS];
  int ncursor_cache = 0;

  uint8_t* state(int i) { return hdr + SLOT0 + i * SLOT_STRIDE; }
  uint8_t* fid(int i) { return hdr + SLOT0 + i * SLOT_STRIDE + 8; }
  uint8_t* ts(int i) { return hdr + SLOT0 + i * SLOT_STRIDE + 16; }
  uint8_t* cursor(int idx) { return hdr + SLOT0 + capacity * SLOT_STRIDE + idx * CURSOR_STRIDE; }
  uint8_t* drops() { return cursor(VPE_MAX_CONSUMERS); }
  uint8_t* evictions() { return drops() + 8; }
  uint8_t* pushed() { return drops() + 16; }
  uint8_t* consumed() { return drops() + 24; }
  uint8_t* slot_ptr(int slot, int label) { return data + ARENA_HDR + offsets[slot * nspecs + label]; }
  int cursor_idx(uint32_t cid) const {
    for (int i = 0; i < ncursor_cache; ++i)
      if (cursor_ids[i] == cid) return cursor_slot[i];
    return -1;
  }
};

static size_t header_region_bytes(int capacity) {
  const size_t need = SLOT0 + (size_t)capacity * SLOT_STRIDE + VPE_MAX_CONSUMERS * CURSOR_STRIDE + 32;
  return std::max<size_t>(4096, align_up(need, 4096));
}

extern "C" {

int64_t vpe_copy_counter(void) { return g_copies.load(); }

int64_t vpe_now_ns(void) {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

void vpe_busy_spin_ns(int64_t ns) {
  if (ns <= 0) return;
  const int64_t end = vpe_now_ns() + ns;
  while (vpe_now_ns() < end) {
  }
}

// ---- AtomicBuffer replacement (_kernels.pyx:56-98): same offset checks, same orders ----
int vpe_atomic_check_base(const void* base, size_t size) {
  if (size > 0 && reinterpret_cast<uintptr_t>(base) % 8 != 0) return VPE_E_VALUE;
  return VPE_OK;
}
static inline bool bad(size_t size, int64_t off, int w) { return off < 0 || off + w > (int64_t)size || off % w; }
int vpe_u32_load(void* b, size_t size, int64_t off, uint32_t* out) {
  if (bad(size, off, 4)) return VPE_E_VALUE;
  *out = ld32(static_cast<uint8_t*>(b) + off);
  return VPE_OK;
}
int vpe_u32_store(void* b, size_t size, int64_t off, uint32_t v) {
  if (bad(size, off, 4)) return VPE_E_VALUE;
  st32(static_cast<uint8_t*>(b) + off, v);
  return VPE_OK;
}
int vpe_u32_cas(void* b, size_t size, int64_t off, uint32_t e, uint32_t d, uint32_t* prev) {
  if (bad(size, off, 4)) return VPE_E_VALUE;
  *prev = cas32(static_cast<uint8_t*>(b) + off, e, d);
  return VPE_OK;
}
int vpe_u64_load(void* b, size_t size, int64_t off, uint64_t* out) {
  if (bad(size, off, 8)) return VPE_E_VALUE;
  *out = ld64(static_cast<uint8_t*>(b) + off);
  return VPE_OK;
}
int vpe_u64_store(void* b, size_t size, int64_t off, uint64_t v) {
  if (bad(size, off, 8)) return VPE_E_VALUE;
  st64(static_cast<uint8_t*>(b) + off, v);
  return VPE_OK;
}
int vpe_u64_add(void* b, size_t size, int64_t off, uint64_t d, uint64_t* prev) {
  if (bad(size, off, 8)) return VPE_E_VALUE;
  *prev = add64(static_cast<uint8_t*>(b) + off, d);
  return VPE_OK;
}

// ---- ring ----
int vpe_ring_destroy(vpe_ring* r) {
  if (!r) return VPE_OK;
  if (r->ready)
    for (int i = 0; i < r->capacity; ++i)
      if (r->ready[i]) cudaEventDestroy(r->ready[i]);
  if (r->done)
    for (int i = 0; i < r->capacity * VPE_MAX_CONSUMERS; ++i)
      if (r->done[i]) cudaEventDestroy(r->done[i]);
  if (r->role) {  // shared ring: unmap (and, for the creator, unlink) the POSIX segments
    if (r->data) {
      if (r->device == VPE_HOST_PLAIN)
        munmap(r->data, r->data_bytes);
      else if (r->role == 2)
        cudaIpcCloseMemHandle(r->data);
      else
        cudaFree(r->data);
    }
    if (r->hdr) munmap(r->hdr, r->hdr_bytes);
    if (r->ipc) munmap(r->ipc, r->ipc_bytes);
    if (r->role == 1) {
      shm_unlink(r->nm_hdr);
      shm_unlink(r->nm_ipc);
      if (r->device == VPE_HOST_PLAIN) shm_unlink(r->nm_dat);
    }
    r->data = nullptr;
    r->hdr = nullptr;
    r->done_valid = nullptr;
  }
  if (r->data) {
    if (r->device == VPE_HOST_PLAIN)
      free(r->data);
    else if (r->device == VPE_HOST_PINNED)
      cudaFreeHost(r->data);
    else
      cudaFree(r->data);
  }
  if (!r->role) free(r->hdr);
  delete[] r->specs;
  delete[] r->nbytes;
  delete[] r->offsets;
  delete[] r->ready;
  delete[] r->done;
  if (!r->role) delete[] r->done_valid;
  delete[] r->pending_evict;
  delete r;
  return VPE_OK;
}

int vpe_ring_create(const vpe_tensor_spec* specs, int32_t nspecs, int32_t capacity, int32_t mode, int32_t device,
                    vpe_ring** out) {
  if (!out) return VPE_E_VALUE;
  if (capacity < 2) return VPE_E_CONFIG;  // channels.py:547-548
  if (nspecs < 1 || !specs) return VPE_E_CONFIG;
  if (mode != VPE_FIFO && mode != VPE_LATEST) return VPE_E_CONFIG;
  for (int i = 0; i < nspecs; ++i) {
    if (itemsize(specs[i].dtype) == 0 || specs[i].rank < 1 || specs[i].rank > 4) return VPE_E_SHAPE;
    for (int d = 0; d < specs[i].rank; ++d)
      if (specs[i].dims[d] <= 0) return VPE_E_SHAPE;
    for (int j = 0; j < i; ++j)
      if (strncmp(specs[i].label, specs[j].label, 64) == 0) return VPE_E_CONFIG;
  }
  vpe_ring* r = new (std::nothrow) vpe_ring();
  if (!r) return VPE_E_RESOURCE;
  r->nspecs = nspecs;
  r->capacity = capacity;
  r->mode = mode;
  r->device = device;
  r->specs = new vpe_tensor_spec[nspecs];
  memcpy(r->specs, specs, sizeof(vpe_tensor_spec) * nspecs);
  r->nbytes = new size_t[nspecs];
  for (int i = 0; i < nspecs; ++i) {
    size_t n = itemsize(specs[i].dtype);
    for (int d = 0; d < specs[i].rank; ++d) n *= (size_t)specs[i].dims[d];
    r->nbytes[i] = n;
  }
  // ArenaLayout.from_specs(specs * capacity): 64-byte aligned, in order (arena.py:114-126)
  r->offsets = new size_t[(size_t)nspecs * capacity];
  size_t cur = 0;
  for (int s = 0; s < capacity; ++s)
    for (int l = 0; l < nspecs; ++l) {
      const size_t off = align_up(cur, ALIGN);
      r->offsets[s * nspecs + l] = off;
      cur = off + r->nbytes[l];
    }
  r->data_bytes = align_up(ARENA_HDR + cur, 4096);
  r->hdr_bytes = header_region_bytes(capacity);
  r->hdr = static_cast<uint8_t*>(aligned_alloc(4096, r->hdr_bytes));
  r->ready = new cudaEvent_t[capacity]();
  r->done = new cudaEvent_t[(size_t)capacity * VPE_MAX_CONSUMERS]();
  r->done_valid = new uint8_t[(size_t)capacity * VPE_MAX_CONSUMERS]();
  r->pending_evict = new int64_t[capacity];
  if (!r->hdr) {
    vpe_ring_destroy(r);
    return VPE_E_RESOURCE;
  }
  memset(r->hdr, 0, r->hdr_bytes);
  memcpy(r->hdr, "PECH1\0", 6);
  r->hdr[6] = (uint8_t)mode;
  uint32_t cap = capacity;
  memcpy(r->hdr + 8, &cap, 4);
  for (int i = 0; i < capacity; ++i) r->pending_evict[i] = -1;
  cudaError_t e = cudaSuccess;
  const bool plain = device == VPE_HOST_PLAIN;
  if (plain) {
    r->data = static_cast<uint8_t*>(aligned_alloc(4096, r->data_bytes));
    if (r->data) memset(r->data, 0, r->data_bytes);
    else e = cudaErrorMemoryAllocation;
  } else if (device == VPE_HOST_PINNED) {
    e = cudaHostAlloc(reinterpret_cast<void**>(&r->data), r->data_bytes, cudaHostAllocPortable);
    if (e == cudaSuccess) memset(r->data, 0, r->data_bytes);
  } else {
    e = cudaMalloc(reinterpret_cast<void**>(&r->data), r->data_bytes);
    if (e == cudaSuccess) e = cudaMemset(r->data, 0, r->data_bytes);
  }
  if (e != cudaSuccess) {
    r->data = nullptr;
    vpe_ring_destroy(r);
    return VPE_E_RESOURCE;
  }
  // PEAR1 region header (arena.py:322-324)
  uint8_t h[ARENA_HDR] = {0};
  memcpy(h, "PEAR1\0", 6);
  uint64_t tb = r->data_bytes;
  memcpy(h + 8, &tb, 8);
  uint32_t nslots = (uint32_t)(nspecs * capacity);
  memcpy(h + 16, &nslots, 4);
  if (plain) {
    memcpy(r->data, h, ARENA_HDR);
    *out = r;
    return VPE_OK;  // host-only ring: no CUDA events, streams must be NULL
  }
  if (cudaMemcpy(r->data, h, ARENA_HDR, cudaMemcpyDefault) != cudaSuccess) {
    vpe_ring_destroy(r);
    return VPE_E_CUDA;
  }
  for (int i = 0; i < capacity; ++i)
    if (cudaEventCreateWithFlags(&r->ready[i], cudaEventDisableTiming) != cudaSuccess) {
      vpe_ring_destroy(r);
      return VPE_E_CUDA;
    }
  for (int i = 0; i < capacity * VPE_MAX_CONSUMERS; ++i)
    if (cudaEventCreateWithFlags(&r->done[i], cudaEventDisableTiming) != cudaSuccess) {
      vpe_ring_destroy(r);
      return VPE_E_CUDA;
    }
  *out = r;
  return VPE_OK;
}

int vpe_ring_header(vpe_ring* r, void** base, size_t* size) {
  if (!r) return VPE_E_VALUE;
  *base = r->hdr;
  *size = r->hdr_bytes;
  return VPE_OK;
}
int vpe_ring_data(vpe_ring* r, void** base, size_t* size) {
  if (!r) return VPE_E_VALUE;
  *base = r->data;
  *size = r->data_bytes;
  return VPE_OK;
}
int vpe_ring_slot_ptr(vpe_ring* r, int32_t slot, int32_t label, void** ptr) {
  if (!r || slot < 0 || slot >= r->capacity) return VPE_E_NOT_FOUND;
  if (label < 0 || label >= r->nspecs) return VPE_E_LABEL;
  *ptr = r->slot_ptr(slot, label);
  return VPE_OK;
}
int vpe_ring_label_offset(vpe_ring* r, int32_t slot, int32_t label, int64_t* off) {
  if (!r || slot < 0 || slot >= r->capacity) return VPE_E_NOT_FOUND;
  if (label < 0 || label >= r->nspecs) return VPE_E_LABEL;
  *off = (int64_t)r->offsets[slot * r->nspecs + label];
  return VPE_OK;
}

// channels.py:311-331 _claim_slot
static int claim_slot(vpe_ring* r, int* slot, int64_t* evicted) {
  for (;;) {
    for (int i = 0; i < r->capacity; ++i)
      if (ld32(r->state(i)) == STATE_FREE && cas32(r->state(i), STATE_FREE, STATE_WRITING) == STATE_FREE) {
        *slot = i;
        *evicted = -1;
        return VPE_OK;
      }
    if (r->mode == VPE_FIFO) return VPE_OVERFLOW_REJECTED;
    int oldest = -1;
    uint64_t oldest_fid = 0;
    for (int i = 0; i < r->capacity; ++i)
      if (ld32(r->state(i)) == STATE_READY) {
        const uint64_t f = ld64(r->fid(i));
        if (oldest < 0 || f < oldest_fid) {
          oldest = i;
          oldest_fid = f;
        }
      }
    if (oldest < 0) return VPE_OVERFLOW_REJECTED;
    if (cas32(r->state(oldest), STATE_READY, STATE_WRITING) == STATE_READY) {
      *slot = oldest;
      *evicted = (int64_t)oldest_fid;
      return VPE_OK;
    }
  }
}

int vpe_ring_claim(vpe_ring* r, uint64_t frame_id, uint64_t capture_ts, void* stream, int32_t* slot,
                   uint64_t* evicted_fid, int32_t* evicted) {
  if (!r || !slot) return VPE_E_VALUE;
  if (frame_id <= r->last_id) return VPE_E_VALUE;  // channels.py:284-285
  if (capture_ts < r->last_ts) return VPE_E_VALUE; // channels.py:286-287
  int s;
  int64_t ev;
  const int rc = claim_slot(r, &s, &ev);
  if (rc == VPE_OVERFLOW_REJECTED) {
    add64(r->drops(), 1);
    add64(r->pushed(), 1);
    return rc;
  }
  st64(r->fid(s), frame_id);
  st64(r->ts(s), capture_ts);
  r->pending_evict[s] = ev;
  if (evicted) *evicted = ev >= 0;
  if (evicted_fid) *evicted_fid = ev >= 0 ? (uint64_t)ev : 0;
  *slot = s;
  // WAR: the new writes must not start before every earlier reader of this slot finished
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (r->device != VPE_HOST_PLAIN)
    for (int c = 0; c < VPE_MAX_CONSUMERS; ++c) {
      const int k = s * VPE_MAX_CONSUMERS + c;
      if (__atomic_load_n(&r->done_valid[k], __ATOMIC_ACQUIRE)) VPE_CUDA_TRY(cudaStreamWaitEvent(st, r->done[k], 0));
    }
  return VPE_OK;
}

int vpe_ring_publish(vpe_ring* r, int32_t slot, void* stream) {
  if (!r || slot < 0 || slot >= r->capacity) return VPE_E_NOT_FOUND;
  if (ld32(r->state(slot)) != STATE_WRITING) return VPE_E_RUNTIME;
  if (r->device != VPE_HOST_PLAIN)
    VPE_CUDA_TRY(cudaEventRecord(r->ready[slot], static_cast<cudaStream_t>(stream)));
  r->last_id = ld64(r->fid(slot));
  r->last_ts = ld64(r->ts(slot));
  st32(r->state(slot), STATE_READY);
  add64(r->pushed(), 1);
  if (r->pending_evict[slot] >= 0) add64(r->evictions(), 1);
  r->pending_evict[slot] = -1;
  return VPE_OK;
}

int vpe_ring_abort(vpe_ring* r, int32_t slot) {
  if (!r || slot < 0 || slot >= r->capacity) return VPE_E_NOT_FOUND;
  r->pending_evict[slot] = -1;
  st32(r->state(slot), STATE_FREE);  // channels.py:299-301
  return VPE_OK;
}

// channels.py:335-358
int vpe_ring_register_consumer(vpe_ring* r, uint32_t cid, int32_t* warn) {
  if (!r) return VPE_E_VALUE;
  if (warn) *warn = 0;
  if (cid < 1 || cid > 0xFFFFFFFEu) return VPE_E_CONFIG;
  int registered = 0;
  for (int idx = 0; idx < VPE_MAX_CONSUMERS; ++idx) {
    const uint32_t cur = ld32(r->cursor(idx));
    if (cur == cid) {
      if (r->cursor_idx(cid) < 0) {
        r->cursor_ids[r->ncursor_cache] = cid;
        r->cursor_slot[r->ncursor_cache++] = idx;
      }
      return VPE_OK;
    }
    if (cur != 0) ++registered;
  }
  for (int idx = 0; idx < VPE_MAX_CONSUMERS; ++idx)
    if (ld32(r->cursor(idx)) == 0 && cas32(r->cursor(idx), 0, cid) == 0) {
      r->cursor_ids[r->ncursor_cache] = cid;
      r->cursor_slot[r->ncursor_cache++] = idx;
      if (warn && r->mode == VPE_LATEST && registered + 2 > r->capacity) *warn = 1;
      return VPE_OK;
    }
  return VPE_E_RESOURCE;
}

int vpe_ring_last_consumed(vpe_ring* r, uint32_t cid, uint64_t* fid) {
  if (!r) return VPE_E_VALUE;
  const int idx = r->cursor_idx(cid);
  if (idx < 0) return VPE_E_NOT_FOUND;
  *fid = ld64(r->cursor(idx) + 8);
  return VPE_OK;
}

// channels.py:423-452
int vpe_ring_acquire_latest(vpe_ring* r, uint32_t cid, void* stream, vpe_lease* lease) {
  if (!r || !lease) return VPE_E_VALUE;
  const int cidx = r->cursor_idx(cid);
  if (cidx < 0) return VPE_E_NOT_FOUND;
  const uint64_t cursor = ld64(r->cursor(cidx) + 8);
  for (;;) {
    int best = -1;
    uint64_t best_fid = cursor;
    uint32_t best_state = 0;
    for (int i = 0; i < r->capacity; ++i) {
      const uint32_t st = ld32(r->state(i));
      if (st >= STATE_READY) {
        const uint64_t f = ld64(r->fid(i));
        if (f > best_fid) {
          best = i;
          best_fid = f;
          best_state = st;
        }
      }
    }
    if (best < 0) return VPE_NO_NEW_DATA;
    uint32_t st = best_state;
    while (st >= STATE_READY) {
      const uint32_t prev = cas32(r->state(best), st, st + 1);
      if (prev == st) {
        lease->slot = best;
        lease->consumer_id = cid;
        lease->frame_id = ld64(r->fid(best));
        lease->capture_ts = ld64(r->ts(best));
        lease->consumed = 0;
        // NULL is the legacy default stream, a valid consumer stream: always order it (RAW)
        if (r->device != VPE_HOST_PLAIN)
          VPE_CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), r->ready[best], 0));
        return VPE_OK;
      }
      st = prev;
    }
  }
}

// channels.py:483-489
static int release_slot(vpe_ring* r, int slot) {
  for (;;) {
    const uint32_t st = ld32(r->state(slot));
    if (st <= STATE_READY) return VPE_E_RUNTIME;
    if (cas32(r->state(slot), st, st - 1) == st) return VPE_OK;
  }
}

static int finish(vpe_ring* r, vpe_lease* lease, void* stream) {
  const int cidx = r->cursor_idx(lease->consumer_id);
  if (cidx < 0) return VPE_E_NOT_FOUND;
  const int k = lease->slot * VPE_MAX_CONSUMERS + cidx;
  if (r->device != VPE_HOST_PLAIN) {  // NULL = legacy default stream, still recorded (WAR)
    VPE_CUDA_TRY(cudaEventRecord(r->done[k], static_cast<cudaStream_t>(stream)));
    __atomic_store_n(&r->done_valid[k], (uint8_t)1, __ATOMIC_RELEASE);
  }
  st64(r->cursor(cidx) + 8, lease->frame_id);  // channels.py:470
  add64(r->consumed(), 1);
  VPE_TRY(release_slot(r, lease->slot));
  lease->consumed = 1;
  return VPE_OK;
}

int vpe_ring_commit(vpe_ring* r, vpe_lease* lease, void* stream) {
  if (!r || !lease) return VPE_E_VALUE;
  if (lease->consumed) return VPE_E_USE_AFTER_CONSUME;
  return finish(r, lease, stream);
}

int vpe_ring_consume(vpe_ring* r, vpe_lease* lease, const int32_t* labels, int32_t nlabels, void* const* dst,
                     void* stream) {
  if (!r || !lease) return VPE_E_VALUE;
  if (lease->consumed) return VPE_E_USE_AFTER_CONSUME;  // channels.py:459-460
  for (int i = 0; i < nlabels; ++i)
    if (labels[i] < 0 || labels[i] >= r->nspecs) return VPE_E_LABEL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < nlabels; ++i) {
    if (r->device == VPE_HOST_PLAIN)
      memcpy(dst[i], r->slot_ptr(lease->slot, labels[i]), r->nbytes[labels[i]]);
    else
      VPE_CUDA_TRY(cudaMemcpyAsync(dst[i], r->slot_ptr(lease->slot, labels[i]), r->nbytes[labels[i]],
                                   cudaMemcpyDefault, st));
    g_copies.fetch_add(1);
  }
  return finish(r, lease, stream);
}

int vpe_ring_release(vpe_ring* r, vpe_lease* lease, void* stream) {
  if (!r || !lease) return VPE_E_VALUE;
  if (lease->consumed) return VPE_OK;  // channels.py:478-479
  if (r->device != VPE_HOST_PLAIN) {
    const int cidx = r->cursor_idx(lease->consumer_id);
    if (cidx >= 0) {
      const int k = lease->slot * VPE_MAX_CONSUMERS + cidx;
      VPE_CUDA_TRY(cudaEventRecord(r->done[k], static_cast<cudaStream_t>(stream)));
      __atomic_store_n(&r->done_valid[k], (uint8_t)1, __ATOMIC_RELEASE);
    }
  }
  VPE_TRY(release_slot(r, lease->slot));
  lease->consumed = 1;
  return VPE_OK;
}

// channels.py:377-421
int vpe_ring_pop(vpe_ring* r, uint32_t cid, void* const* dst, int32_t dst_on_host, void* stream, vpe_lease* env) {
  if (!r) return VPE_E_VALUE;
  if (r->mode != VPE_FIFO) return VPE_E_CONFIG;
  const int cidx = r->cursor_idx(cid);
  if (cidx < 0) return VPE_E_NOT_FOUND;
  for (;;) {
    int best = -1;
    uint64_t best_fid = 0;
    for (int i = 0; i < r->capacity; ++i)
      if (ld32(r->state(i)) == STATE_READY) {
        const uint64_t f = ld64(r->fid(i));
        if (best < 0 || f < best_fid) {
          best = i;
          best_fid = f;
        }
      }
    if (best < 0) return VPE_NO_NEW_DATA;
    if (cas32(r->state(best), STATE_READY, STATE_READY + 1) != STATE_READY) continue;
    const uint64_t fid = ld64(r->fid(best));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!dst_on_host && r->device != VPE_HOST_PLAIN) {
      VPE_CUDA_TRY(cudaStreamWaitEvent(st, r->ready[best], 0));
      for (int l = 0; l < r->nspecs; ++l) {
        VPE_CUDA_TRY(cudaMemcpyAsync(dst[l], r->slot_ptr(best, l), r->nbytes[l], cudaMemcpyDefault, st));
        g_copies.fetch_add(1);
      }
      const int k = best * VPE_MAX_CONSUMERS + cidx;
      VPE_CUDA_TRY(cudaEventRecord(r->done[k], st));
      __atomic_store_n(&r->done_valid[k], (uint8_t)1, __ATOMIC_RELEASE);
    } else {
      // host consumer: wait for the producer's writes, then copy on the host
      if (r->device != VPE_HOST_PLAIN) VPE_CUDA_TRY(cudaEventSynchronize(r->ready[best]));
      for (int l = 0; l < r->nspecs; ++l) {
        if (r->device == VPE_HOST_PINNED || r->device == VPE_HOST_PLAIN)
          memcpy(dst[l], r->slot_ptr(best, l), r->nbytes[l]);
        else
          VPE_CUDA_TRY(cudaMemcpy(dst[l], r->slot_ptr(best, l), r->nbytes[l], cudaMemcpyDefault));
        g_copies.fetch_add(1);
      }
    }
    if (env) {
      env->slot = best;
      env->consumer_id = cid;
      env->frame_id = fid;
      env->capture_ts = ld64(r->ts(best));
      env->consumed = 1;
    }
    st64(r->cursor(cidx) + 8, fid);
    add64(r->consumed(), 1);
    st32(r->state(best), STATE_FREE);
    return VPE_OK;
  }
}

int vpe_ring_counters(vpe_ring* r, vpe_counters* c) {
  if (!r || !c) return VPE_E_VALUE;
  uint64_t resident = 0;
  for (int i = 0; i < r->capacity; ++i)
    if (ld32(r->state(i)) >= STATE_READY) ++resident;
  c->pushed = ld64(r->pushed());
  c->producer_drops = ld64(r->drops());
  c->evictions = ld64(r->evictions());
  c->consumed = ld64(r->consumed());
  c->resident = resident;
  return VPE_OK;
}

int vpe_ring_slot_state(vpe_ring* r, int32_t slot, uint32_t* state, uint64_t* fid) {
  if (!r || slot < 0 || slot >= r->capacity) return VPE_E_NOT_FOUND;
  *state = ld32(r->state(slot));
  *fid = ld64(r->fid(slot));
  return VPE_OK;
}


// ---------------------------------------------------------------------------------------------
// Cross-process rings (PAPER.md:95-121 runs every head in its own process).
// The reference shares its arena and channel header through POSIX shared memory
// (arena.py:285-344, channels.py:537-594). Here the PECH1 control block lives in a POSIX
// segment "<name>-c" (state words keep the same acquire/release CAS protocol across processes),
// the HBM slot arena is exported with cudaIpcGetMemHandle, and the ready / done events are
// created cudaEventInterprocess and exported with cudaIpcGetEventHandle; all handles plus the
// shared done-valid flags sit in "<name>-x". A plain-host ring keeps its data in "<name>-d".
namespace {
constexpr char IPC_MAGIC[8] = {'P', 'E', 'I', 'P', 'C', '1', 0, 0};
struct IpcHead {
  char magic[8];
  int32_t device, capacity, nspecs, mode;
  uint64_t data_bytes, hdr_bytes;
  cudaIpcMemHandle_t mem;
};
size_t ipc_layout(int capacity, int nspecs, size_t* off_specs, size_t* off_ready, size_t* off_done,
                  size_t* off_valid) {
  size_t o = align_up(sizeof(IpcHead), 64);
  *off_specs = o;
  o += align_up(sizeof(vpe_tensor_spec) * (size_t)nspecs, 64);
  *off_ready = o;
  o += sizeof(cudaIpcEventHandle_t) * (size_t)capacity;
  *off_done = o;
  o += sizeof(cudaIpcEventHandle_t) * (size_t)capacity * VPE_MAX_CONSUMERS;
  *off_valid = o;
  o += (size_t)capacity * VPE_MAX_CONSUMERS;
  return align_up(o, 4096);
}
int shm_map(const char* name, size_t bytes, bool create, void** base, size_t* mapped) {
  const int fd = shm_open(name, create ? (O_CREAT | O_EXCL | O_RDWR) : O_RDWR, 0600);
  if (fd < 0) return errno == EEXIST ? VPE_E_ALREADY_EXISTS : (errno == ENOENT ? VPE_E_NOT_FOUND : VPE_E_RESOURCE);
  if (create) {
    if (ftruncate(fd, (off_t)bytes) != 0) {
      close(fd);
      shm_unlink(name);
      return VPE_E_RESOURCE;
    }
  } else {
    struct stat st;
    if (fstat(fd, &st) != 0 || (size_t)st.st_size < 64) {
      close(fd);
      return VPE_E_CORRUPT_HANDLE;
    }
    bytes = (size_t)st.st_size;
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    if (create) shm_unlink(name);
    return VPE_E_RESOURCE;
  }
  *base = p;
  *mapped = bytes;
  return VPE_OK;
}
// segment names follow the reference's "<namespace>.<region>" convention (arena.py:163-165,
// channels.py:568 "<name>-c"), so shm_census / clean_namespace see them
void shm_names(vpe_ring* r, const char* name) {
  snprintf(r->nm_hdr, sizeof(r->nm_hdr), "/%s-c", name);
  snprintf(r->nm_ipc, sizeof(r->nm_ipc), "/%s-x", name);
  snprintf(r->nm_dat, sizeof(r->nm_dat), "/%s-d", name);
}
}  // namespace

int vpe_ring_create_shared(const vpe_tensor_spec* specs, int32_t nspecs, int32_t capacity, int32_t mode,
                           int32_t device, const char* name, vpe_ring** out) {
  if (!out || !name || !name[0] || strlen(name) > 150 || strchr(name, '/')) return VPE_E_CONFIG;
  if (device == VPE_HOST_PINNED) return VPE_E_CONFIG;  // pinned host memory is not exportable here
  // build the layout and CUDA objects privately first, then move the control block into shm
  vpe_ring* r = nullptr;
  VPE_TRY(vpe_ring_create(specs, nspecs, capacity, mode, device, &r));
  shm_names(r, name);
  size_t o_specs, o_ready, o_done, o_valid;
  const size_t ipc_bytes = ipc_layout(capacity, nspecs, &o_specs, &o_ready, &o_done, &o_valid);
  void* hdr = nullptr;
  void* ipc = nullptr;
  size_t hdr_map = 0, ipc_map = 0;
  int rc = shm_map(r->nm_hdr, r->hdr_bytes, true, &hdr, &hdr_map);
  if (rc) {
    vpe_ring_destroy(r);
    return rc;
  }
  rc = shm_map(r->nm_ipc, ipc_bytes, true, &ipc, &ipc_map);
  if (rc) {
    munmap(hdr, hdr_map);
    shm_unlink(r->nm_hdr);
    vpe_ring_destroy(r);
    return rc;
  }
  memcpy(hdr, r->hdr, r->hdr_bytes);
  free(r->hdr);
  r->hdr = static_cast<uint8_t*>(hdr);
  r->ipc = static_cast<uint8_t*>(ipc);
  r->ipc_bytes = ipc_map;
  memset(r->ipc, 0, ipc_map);
  delete[] r->done_valid;
  r->done_valid = r->ipc + o_valid;
  r->role = 1;
  IpcHead* h = reinterpret_cast<IpcHead*>(r->ipc);
  memcpy(h->magic, IPC_MAGIC, 8);
  h->device = device;
  h->capacity = capacity;
  h->nspecs = nspecs;
  h->mode = mode;
  h->data_bytes = r->data_bytes;
  h->hdr_bytes = r->hdr_bytes;
  memcpy(r->ipc + o_specs, specs, sizeof(vpe_tensor_spec) * (size_t)nspecs);
  if (device == VPE_HOST_PLAIN) {
    void* dat = nullptr;
    size_t dat_map = 0;
    if ((rc = shm_map(r->nm_dat, r->data_bytes, true, &dat, &dat_map))) {
      vpe_ring_destroy(r);
      return rc;
    }
    memcpy(dat, r->data, r->data_bytes);
    free(r->data);
    r->data = static_cast<uint8_t*>(dat);
    *out = r;
    return VPE_OK;
  }
  // device ring: export the arena and interprocess events
  if (cudaIpcGetMemHandle(&h->mem, r->data) != cudaSuccess) {
    vpe_ring_destroy(r);
    return VPE_E_CUDA;
  }
  auto remake = [&](cudaEvent_t* e, cudaIpcEventHandle_t* eh) -> bool {
    cudaEventDestroy(*e);
    *e = nullptr;
    return cudaEventCreateWithFlags(e, cudaEventDisableTiming | cudaEventInterprocess) == cudaSuccess &&
           cudaIpcGetEventHandle(eh, *e) == cudaSuccess;
  };
  auto* ready_h = reinterpret_cast<cudaIpcEventHandle_t*>(r->ipc + o_ready);
  auto* done_h = reinterpret_cast<cudaIpcEventHandle_t*>(r->ipc + o_done);
  for (int i = 0; i < capacity; ++i)
    if (!remake(&r->ready[i], &ready_h[i])) {
      vpe_ring_destroy(r);
      return VPE_E_CUDA;
    }
  for (int i = 0; i < capacity * VPE_MAX_CONSUMERS; ++i)
    if (!remake(&r->done[i], &done_h[i])) {
      vpe_ring_destroy(r);
      return VPE_E_CUDA;
    }
  *out = r;
  return VPE_OK;
}

int vpe_ring_attach(const char* name, vpe_ring** out) {
  if (!out || !name || !name[0] || strlen(name) > 150 || strchr(name, '/')) return VPE_E_CONFIG;
  vpe_ring* r = new (std::nothrow) vpe_ring();
  if (!r) return VPE_E_RESOURCE;
  shm_names(r, name);
  r->role = 2;
  void* ipc = nullptr;
  size_t ipc_map = 0;
  int rc = shm_map(r->nm_ipc, 0, false, &ipc, &ipc_map);
  if (rc) {
    delete r;
    return rc;
  }
  r->ipc = static_cast<uint8_t*>(ipc);
  r->ipc_bytes = ipc_map;
  const IpcHead* h = reinterpret_cast<const IpcHead*>(r->ipc);
  if (memcmp(h->magic, IPC_MAGIC, 8) != 0 || h->capacity < 2 || h->nspecs < 1) {
    vpe_ring_destroy(r);
    return VPE_E_CORRUPT_HANDLE;
  }
  size_t o_specs, o_ready, o_done, o_valid;
  if (ipc_layout(h->capacity, h->nspecs, &o_specs, &o_ready, &o_done, &o_valid) > ipc_map) {
    vpe_ring_destroy(r);
    return VPE_E_CORRUPT_HANDLE;
  }
  // rebuild the layout from the published specs (same code path as the creator)
  vpe_ring* tmp = nullptr;
  const int dev_for_layout = VPE_HOST_PLAIN;  // layout only: no allocation of CUDA objects
  (void)dev_for_layout;
  r->nspecs = h->nspecs;
  r->capacity = h->capacity;
  r->mode = h->mode;
  r->device = h->device;
  r->specs = new vpe_tensor_spec[r->nspecs];
  memcpy(r->specs, r->ipc + o_specs, sizeof(vpe_tensor_spec) * (size_t)r->nspecs);
  r->nbytes = new size_t[r->nspecs];
  for (int i = 0; i < r->nspecs; ++i) {
    size_t n = itemsize(r->specs[i].dtype);
    for (int d = 0; d < r->specs[i].rank; ++d) n *= (size_t)r->specs[i].dims[d];
    r->nbytes[i] = n;
  }
  r->offsets = new size_t[(size_t)r->nspecs * r->capacity];
  size_t cur = 0;
  for (int sl = 0; sl < r->capacity; ++sl)
    for (int l = 0; l < r->nspecs; ++l) {
      const size_t off = align_up(cur, ALIGN);
      r->offsets[sl * r->nspecs + l] = off;
      cur = off + r->nbytes[l];
    }
  (void)tmp;
  r->data_bytes = h->data_bytes;
  r->pending_evict = new int64_t[r->capacity];
  for (int i = 0; i < r->capacity; ++i) r->pending_evict[i] = -1;
  r->ready = new cudaEvent_t[r->capacity]();
  r->done = new cudaEvent_t[(size_t)r->capacity * VPE_MAX_CONSUMERS]();
  r->done_valid = r->ipc + o_valid;
  void* hdr = nullptr;
  size_t hdr_map = 0;
  if ((rc = shm_map(r->nm_hdr, 0, false, &hdr, &hdr_map))) {
    vpe_ring_destroy(r);
    return rc;
  }
  r->hdr = static_cast<uint8_t*>(hdr);
  r->hdr_bytes = hdr_map;
  if (memcmp(r->hdr, "PECH1\0", 6) != 0 || r->hdr[6] != (uint8_t)r->mode) {
    vpe_ring_destroy(r);
    return VPE_E_CORRUPT_HANDLE;
  }
  if (r->device == VPE_HOST_PLAIN) {
    void* dat = nullptr;
    size_t dat_map = 0;
    if ((rc = shm_map(r->nm_dat, 0, false, &dat, &dat_map))) {
      vpe_ring_destroy(r);
      return rc;
    }
    r->data = static_cast<uint8_t*>(dat);
    *out = r;
    return VPE_OK;
  }
  void* dptr = nullptr;
  if (cudaSetDevice(r->device) != cudaSuccess ||
      cudaIpcOpenMemHandle(&dptr, h->mem, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    vpe_ring_destroy(r);
    return VPE_E_CUDA;
  }
  r->data = static_cast<uint8_t*>(dptr);
  auto* ready_h = reinterpret_cast<cudaIpcEventHandle_t*>(r->ipc + o_ready);
  auto* done_h = reinterpret_cast<cudaIpcEventHandle_t*>(r->ipc + o_done);
  for (int i = 0; i < r->capacity; ++i)
    if (cudaIpcOpenEventHandle(&r->ready[i], ready_h[i]) != cudaSuccess) {
      vpe_ring_destroy(r);
      return VPE_E_CUDA;
    }
  for (int i = 0; i < r->capacity * VPE_MAX_CONSUMERS; ++i)
    if (cudaIpcOpenEventHandle(&r->done[i], done_h[i]) != cudaSuccess) {
      vpe_ring_destroy(r);
      return VPE_E_CUDA;
    }
  *out = r;
  return VPE_OK;
}


// ---------------------------------------------------------------------------------------------
// Shareable regions: the reference's create_region / attach_region (arena.py:285-313) with the
// bytes in HBM (CUDA IPC export) or in POSIX shared memory (VPE_HOST_PLAIN). A POSIX segment
// "/<namespace>.<region>" always exists for a region: for a host region it holds the bytes, for
// a device region a descriptor {magic, device, bytes, cudaIpcMemHandle}.
struct vpe_region {
  int32_t device = 0;
  int role = 0;  // 1 creator, 2 attached
  size_t bytes = 0;
  uint8_t* base = nullptr;
  void* seg = nullptr;
  size_t seg_bytes = 0;
  char nm[192] = {0};
};
namespace {
constexpr char REG_MAGIC[8] = {'P', 'E', 'R', 'E', 'G', '1', 0, 0};
struct RegDesc {
  char magic[8];
  int32_t device, pad;
  uint64_t bytes;
  cudaIpcMemHandle_t mem;
};
bool region_name_ok(const char* name) {
  return name && name[0] && strlen(name) <= 150 && !strchr(name, '/');
}
}  // namespace

int vpe_region_destroy(vpe_region* g, int32_t unlink) {
  if (!g) return VPE_OK;
  if (g->device >= 0 && g->base) {
    if (g->role == 2)
      cudaIpcCloseMemHandle(g->base);
    else
      cudaFree(g->base);
  }
  if (g->seg) munmap(g->seg, g->seg_bytes);
  if (unlink && g->nm[0]) shm_unlink(g->nm);
  delete g;
  return VPE_OK;
}

int vpe_region_create(const char* name, uint64_t nbytes, int32_t device, vpe_region** out) {
  if (!out || !region_name_ok(name) || nbytes == 0) return VPE_E_CONFIG;
  if (device == VPE_HOST_PINNED) return VPE_E_CONFIG;  // pinned host memory is not shareable here
  vpe_region* g = new (std::nothrow) vpe_region();
  if (!g) return VPE_E_RESOURCE;
  snprintf(g->nm, sizeof(g->nm), "/%s", name);
  g->device = device;
  g->bytes = nbytes;
  g->role = 1;
  const bool host = device == VPE_HOST_PLAIN;
  int rc = shm_map(g->nm, host ? nbytes : sizeof(RegDesc), true, &g->seg, &g->seg_bytes);
  if (rc) {
    g->nm[0] = 0;  // never unlink a segment we did not create (AlreadyExists)
    vpe_region_destroy(g, 0);
    return rc;
  }
  memset(g->seg, 0, g->seg_bytes);  // zero-initialised
  if (host) {
    g->base = static_cast<uint8_t*>(g->seg);
    *out = g;
    return VPE_OK;
  }
  RegDesc* d = static_cast<RegDesc*>(g->seg);
  if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(reinterpret_cast<void**>(&g->base), nbytes) != cudaSuccess ||
      cudaMemset(g->base, 0, nbytes) != cudaSuccess || cudaIpcGetMemHandle(&d->mem, g->base) != cudaSuccess) {
    cudaGetLastError();
    vpe_region_destroy(g, 1);
    return VPE_E_RESOURCE;
  }
  d->device = device;
  d->bytes = nbytes;
  memcpy(d->magic, REG_MAGIC, 8);  // published last: attachers see a complete descriptor
  *out = g;
  return VPE_OK;
}

int vpe_region_attach(const char* name, uint64_t expect_bytes, vpe_region** out) {
  if (!out || !region_name_ok(name)) return VPE_E_CONFIG;
  vpe_region* g = new (std::nothrow) vpe_region();
  if (!g) return VPE_E_RESOURCE;
  snprintf(g->nm, sizeof(g->nm), "/%s", name);
  g->role = 2;
  const int rc = shm_map(g->nm, 0, false, &g->seg, &g->seg_bytes);
  if (rc) {
    g->nm[0] = 0;
    vpe_region_destroy(g, 0);
    return rc;
  }
  const RegDesc* d = static_cast<const RegDesc*>(g->seg);
  const bool dev = g->seg_bytes >= sizeof(RegDesc) && memcmp(d->magic, REG_MAGIC, 8) == 0;
  if (!dev) {  // a host region: the segment is the bytes
    g->device = VPE_HOST_PLAIN;
    g->bytes = g->seg_bytes;
    g->base = static_cast<uint8_t*>(g->seg);
  } else {
    g->device = d->device;
    g->bytes = d->bytes;
    void* p = nullptr;
    if (cudaSetDevice(d->device) != cudaSuccess ||
        cudaIpcOpenMemHandle(&p, d->mem, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      g->nm[0] = 0;
      vpe_region_destroy(g, 0);
      return VPE_E_RESOURCE;
    }
    g->base = static_cast<uint8_t*>(p);
  }
  if (g->bytes < expect_bytes) {  // attach_region: handle larger than the mapping (arena.py:310-312)
    g->nm[0] = 0;
    vpe_region_destroy(g, 0);
    return VPE_E_CORRUPT_HANDLE;
  }
  *out = g;
  return VPE_OK;
}

int vpe_region_info(vpe_region* g, void** base, uint64_t* bytes, int32_t* device) {
  if (!g) return VPE_E_VALUE;
  if (base) *base = g->base;
  if (bytes) *bytes = g->bytes;
  if (device) *device = g->device;
  return VPE_OK;
}

// copy_out (arena.py:367-373): the single permitted copy, stream-ordered for device memory;
// host_sync != 0 returns only when the bytes are in dst
int vpe_copy_out(void* dst, const void* src, uint64_t nbytes, void* stream, int32_t host_sync) {
  if ((!dst || !src) && nbytes) return VPE_E_VALUE;
  cudaPointerAttributes a{}, b{};
  const bool dev_src = cudaPointerGetAttributes(&a, src) == cudaSuccess && a.type == cudaMemoryTypeDevice;
  const bool dev_dst = cudaPointerGetAttributes(&b, dst) == cudaSuccess && b.type == cudaMemoryTypeDevice;
  cudaGetLastError();
  if (!dev_src && !dev_dst) {
    memcpy(dst, src, nbytes);
  } else {
    VPE_CUDA_TRY(cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
    if (host_sync) VPE_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  }
  g_copies.fetch_add(1);
  return VPE_OK;
}

}  // extern "C"
