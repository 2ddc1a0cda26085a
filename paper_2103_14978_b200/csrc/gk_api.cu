// gk_api.cu -- the C ABI (include/gatekeeper.h): host-side validation, then the
// launches.  No global mutable state apart from the thread-local last CUDA error.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/gatekeeper.h"
#include "gk_kernels.cuh"

namespace gk {
int launch_edit_distance(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                         int len, int32_t* dist, cudaStream_t stream);
int launch_accuracy(const uint32_t* accept, int64_t astride, const uint8_t* errc, int64_t estride,
                    const int32_t* dist, int64_t n, const int32_t* e_list, int rows,
                    unsigned long long* counts, cudaStream_t stream);
int launch_pack_planes(const uint8_t* rows, int64_t n_rows, int64_t len, int64_t stride,
                       uint32_t* planes, cudaStream_t stream);
int launch_gather_windows(const uint32_t* planes, int64_t nbases, const int64_t* offsets, int64_t n,
                          int len, uint32_t* packed, uint32_t* undef, cudaStream_t stream);
}  // namespace gk

static thread_local int g_last_cuda_error = 0;

namespace gk {
void ensure_func_attr(const void* f, cudaFuncAttribute attr, int value) {
  struct Entry {
    int dev;
    const void* f;
    int attr;
    int value;
  };
  static thread_local Entry seen[256];
  static thread_local int nseen = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  for (int i = 0; i < nseen; ++i) {
    Entry& e = seen[i];
    if (e.dev == dev && e.f == f && e.attr == (int)attr) {
      if (e.value != value) {
        cudaFuncSetAttribute(f, attr, value);
        e.value = value;
      }
      return;
    }
  }
  cudaFuncSetAttribute(f, attr, value);
  if (nseen < 256) seen[nseen++] = Entry{dev, f, (int)attr, value};
}
}  // namespace gk
static std::atomic<uint64_t> g_launches{0};

namespace gk {
void count_launch(int k) { g_launches.fetch_add((uint64_t)k, std::memory_order_relaxed); }
}  // namespace gk

static int cuda_status(cudaError_t err) {
  if (err == cudaSuccess) return GK_OK;
  g_last_cuda_error = (int)err;
  return GK_ERR_CUDA;
}

static int after_launch() { return cuda_status(cudaGetLastError()); }

static bool aligned(const void* p, uintptr_t a) {
  return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0;
}

extern "C" {

int gk_version(void) { return 10000; }

const char* gk_status_string(int status) {
  switch (status) {
    case GK_OK: return "ok";
    case GK_ERR_ARG: return "invalid argument";
    case GK_ERR_LEN: return "len outside [1, GK_MAX_LEN]";
    case GK_ERR_E: return "e outside [0, len)";
    case GK_ERR_ALIGN: return "misaligned buffer";
    case GK_ERR_WORKSPACE: return "workspace missing or too small";
    case GK_ERR_CUDA: return "CUDA error (see gk_last_cuda_error)";
    default: return "unknown status";
  }
}

int gk_last_cuda_error(void) { return g_last_cuda_error; }

uint64_t gk_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

size_t gk_packed_words(int64_t n_seqs, int32_t len) {
  if (n_seqs <= 0 || len <= 0) return 0;
  return (size_t)((n_seqs + GK_TILE - 1) / GK_TILE) * (size_t)len * 64u;
}

size_t gk_undef_words(int64_t n_seqs) {
  if (n_seqs <= 0) return 0;
  return (size_t)((n_seqs + GK_TILE - 1) / GK_TILE) * 32u;
}

size_t gk_result_words(int64_t n_pairs) {
  if (n_pairs <= 0) return 0;
  return (size_t)((n_pairs + 31) / 32);
}

static int check_ascii(const void* p, int64_t n, int32_t len, int64_t stride) {
  if (n < 0) return GK_ERR_ARG;
  if (len < 1 || len > GK_MAX_LEN) return GK_ERR_LEN;
  if (stride < len || stride > GK_MAX_STRIDE) return GK_ERR_ARG;
  if (n > 0 && p == nullptr) return GK_ERR_ARG;
  return GK_OK;
}

int gk_encode(const uint8_t* d_seqs, int64_t n_seqs, int32_t len, int64_t stride,
              uint32_t* d_packed, uint32_t* d_undef, void* stream) {
  int rc = check_ascii(d_seqs, n_seqs, len, stride);
  if (rc) return rc;
  if (n_seqs == 0) return GK_OK;
  if (!d_packed || !d_undef) return GK_ERR_ARG;
  if (!aligned(d_packed, 16) || !aligned(d_undef, 4)) return GK_ERR_ALIGN;
  gk::launch_encode(d_seqs, n_seqs, len, stride, d_packed, d_undef, (cudaStream_t)stream);
  return after_launch();
}

int gk_filter_ex(const uint32_t* d_reads_packed, const uint32_t* d_refs_packed,
                 const uint32_t* d_read_undef, const uint32_t* d_ref_undef, int64_t n_pairs,
                 int32_t len, int32_t e, uint32_t* d_accept_bits, uint8_t* d_errcount,
                 int32_t flags, void* stream) {
  if (n_pairs < 0) return GK_ERR_ARG;
  if (len < 1 || len > GK_MAX_LEN) return GK_ERR_LEN;
  if (e < 0 || e >= len) return GK_ERR_E;
  if (n_pairs == 0) return GK_OK;
  if (!d_reads_packed || !d_refs_packed || !d_read_undef || !d_ref_undef || !d_accept_bits)
    return GK_ERR_ARG;
  if (!aligned(d_reads_packed, 16) || !aligned(d_refs_packed, 16) || !aligned(d_read_undef, 4) ||
      !aligned(d_ref_undef, 4) || !aligned(d_accept_bits, 4))
    return GK_ERR_ALIGN;
  gk::launch_filter(d_reads_packed, d_refs_packed, d_read_undef, d_ref_undef, n_pairs, len, e,
                    d_accept_bits, d_errcount, flags & (GK_FLAG_GENERIC | GK_FLAG_NO_EDGE_FIX | GK_FLAG_BLOCKED),
                    (cudaStream_t)stream);
  return after_launch();
}

int gk_filter(const uint32_t* d_reads_packed, const uint32_t* d_refs_packed,
              const uint32_t* d_read_undef, const uint32_t* d_ref_undef, int64_t n_pairs,
              int32_t len, int32_t e, uint32_t* d_accept_bits, uint8_t* d_errcount,
              void* stream) {
  return gk_filter_ex(d_reads_packed, d_refs_packed, d_read_undef, d_ref_undef, n_pairs, len, e,
                      d_accept_bits, d_errcount, 0, stream);
}

int gk_filter_sweep(const uint32_t* d_reads_packed, const uint32_t* d_refs_packed,
                    const uint32_t* d_read_undef, const uint32_t* d_ref_undef, int64_t n_pairs,
                    int32_t len, int32_t e_max, uint32_t* d_accept_bits, uint8_t* d_errcount,
                    int32_t flags, void* stream) {
  if (n_pairs < 0) return GK_ERR_ARG;
  if (len < 1 || len > GK_MAX_LEN) return GK_ERR_LEN;
  if (e_max < 0 || e_max >= len) return GK_ERR_E;
  if (n_pairs == 0) return GK_OK;
  if (!d_reads_packed || !d_refs_packed || !d_read_undef || !d_ref_undef || !d_accept_bits)
    return GK_ERR_ARG;
  if (!aligned(d_reads_packed, 16) || !aligned(d_refs_packed, 16) || !aligned(d_read_undef, 4) ||
      !aligned(d_ref_undef, 4) || !aligned(d_accept_bits, 4))
    return GK_ERR_ALIGN;
  gk::launch_filter_sweep(d_reads_packed, d_refs_packed, d_read_undef, d_ref_undef, n_pairs, len,
                          e_max, d_accept_bits, d_errcount, flags & GK_FLAG_NO_EDGE_FIX,
                          (cudaStream_t)stream);
  return after_launch();
}

int gk_filter_ascii(const uint8_t* d_reads, const uint8_t* d_refs, int64_t stride,
                    int64_t n_pairs, int32_t len, int32_t e, uint32_t* d_accept_bits,
                    uint8_t* d_errcount, void* stream) {
  int rc = check_ascii(d_reads, n_pairs, len, stride);
  if (rc) return rc;
  if (n_pairs > 0 && d_refs == nullptr) return GK_ERR_ARG;
  if (e < 0 || e >= len) return GK_ERR_E;
  if (n_pairs == 0) return GK_OK;
  if (!d_accept_bits) return GK_ERR_ARG;
  if (!aligned(d_accept_bits, 4)) return GK_ERR_ALIGN;
  gk::launch_filter_ascii(d_reads, d_refs, stride, n_pairs, len, e, d_accept_bits, d_errcount,
                          (cudaStream_t)stream);
  return after_launch();
}

int gk_filter_ascii_sweep(const uint8_t* d_reads, const uint8_t* d_refs, int64_t stride,
                          int64_t n_pairs, int32_t len, int32_t e_max, uint32_t* d_accept_bits,
                          uint8_t* d_errcount, void* stream) {
  int rc = check_ascii(d_reads, n_pairs, len, stride);
  if (rc) return rc;
  if (n_pairs > 0 && d_refs == nullptr) return GK_ERR_ARG;
  if (e_max < 0 || e_max >= len) return GK_ERR_E;
  if (n_pairs == 0) return GK_OK;
  if (!d_accept_bits) return GK_ERR_ARG;
  if (!aligned(d_accept_bits, 4)) return GK_ERR_ALIGN;
  if (!aligned(d_reads, 16) || !aligned(d_refs, 16)) return GK_ERR_ALIGN;
  if (!gk::launch_fused(d_reads, d_refs, stride, n_pairs, len, e_max, true, d_accept_bits,
                        d_errcount, (cudaStream_t)stream))
    return GK_ERR_LEN;  // the tile does not fit in shared memory: gk_encode + gk_filter_sweep
  return after_launch();
}

size_t gk_compact_workspace_bytes(int64_t n_pairs) {
  return gk::compact_workspace_bytes(n_pairs < 0 ? 0 : n_pairs);
}

int gk_compact(const uint32_t* d_accept_bits, int64_t n_pairs, uint32_t* d_idx,
               uint64_t* d_n_acc, void* d_ws, size_t ws_bytes, void* stream) {
  if (n_pairs < 0 || n_pairs >= ((int64_t)1 << 32)) return GK_ERR_ARG;
  if (!d_n_acc) return GK_ERR_ARG;
  if (!aligned(d_n_acc, 8)) return GK_ERR_ALIGN;
  if (n_pairs == 0) return cuda_status(cudaMemsetAsync(d_n_acc, 0, 8, (cudaStream_t)stream));
  if (!d_accept_bits) return GK_ERR_ARG;
  if (!aligned(d_accept_bits, 4) || (d_idx && !aligned(d_idx, 4))) return GK_ERR_ALIGN;
  if (!d_ws || ws_bytes < gk::compact_workspace_bytes(n_pairs)) return GK_ERR_WORKSPACE;
  gk::launch_compact(d_accept_bits, n_pairs, d_idx, d_n_acc, d_ws, (cudaStream_t)stream);
  return after_launch();
}

size_t gk_compact_rows_workspace_bytes(int64_t n_pairs, int32_t n_rows) {
  return gk::compact_workspace_bytes(n_pairs < 0 ? 0 : n_pairs, n_rows < 1 ? 1 : n_rows);
}

int gk_compact_rows(const uint32_t* d_accept_bits, int32_t n_rows, int64_t bits_row_stride,
                    int64_t n_pairs, uint32_t* d_idx, int64_t idx_row_stride, uint64_t* d_n_acc,
                    void* d_ws, size_t ws_bytes, void* stream) {
  if (n_pairs < 0 || n_pairs >= ((int64_t)1 << 32) || n_rows < 0 || n_rows > 65535)
    return GK_ERR_ARG;
  if (n_rows == 0) return GK_OK;
  if (!d_n_acc) return GK_ERR_ARG;
  if (!aligned(d_n_acc, 8)) return GK_ERR_ALIGN;
  if (n_pairs == 0)
    return cuda_status(cudaMemsetAsync(d_n_acc, 0, 8 * (size_t)n_rows, (cudaStream_t)stream));
  if (!d_accept_bits) return GK_ERR_ARG;
  if (n_rows > 1 && bits_row_stride < (int64_t)gk_result_words(n_pairs)) return GK_ERR_ARG;
  if (d_idx && n_rows > 1 && idx_row_stride < n_pairs) return GK_ERR_ARG;
  if (!aligned(d_accept_bits, 4) || (d_idx && !aligned(d_idx, 4))) return GK_ERR_ALIGN;
  if (!d_ws || ws_bytes < gk::compact_workspace_bytes(n_pairs, n_rows)) return GK_ERR_WORKSPACE;
  gk::launch_compact(d_accept_bits, n_pairs, d_idx, d_n_acc, d_ws, (cudaStream_t)stream, n_rows,
                     bits_row_stride, idx_row_stride);
  return after_launch();
}

size_t gk_plane_words(int64_t n_bases) {
  if (n_bases < 0) return 0;
  return (size_t)((n_bases + 31) / 32 + 1);
}

int gk_pack_planes(const uint8_t* d_rows, int64_t n_rows, int64_t len, int64_t stride,
                   uint32_t* d_planes, void* stream) {
  if (n_rows < 0 || stride < len) return GK_ERR_ARG;
  if (len < 1) return GK_ERR_LEN;
  if (n_rows == 0) return GK_OK;
  if (!d_rows || !d_planes) return GK_ERR_ARG;
  if (!aligned(d_planes, 16)) return GK_ERR_ALIGN;
  gk::launch_pack_planes(d_rows, n_rows, len, stride, d_planes, (cudaStream_t)stream);
  return after_launch();
}

int gk_gather_windows(const uint32_t* d_planes, int64_t n_bases, const int64_t* d_offsets,
                      int64_t n_pairs, int32_t len, uint32_t* d_packed, uint32_t* d_undef,
                      void* stream) {
  if (n_pairs < 0 || n_bases < 0) return GK_ERR_ARG;
  if (len < 1 || len > GK_MAX_LEN) return GK_ERR_LEN;
  if (n_pairs == 0) return GK_OK;
  if (!d_planes || !d_offsets || !d_packed || !d_undef) return GK_ERR_ARG;
  if (!aligned(d_packed, 16) || !aligned(d_undef, 4) || !aligned(d_offsets, 8) ||
      !aligned(d_planes, 16))
    return GK_ERR_ALIGN;
  gk::launch_gather_windows(d_planes, n_bases, d_offsets, n_pairs, len, d_packed, d_undef,
                            (cudaStream_t)stream);
  return after_launch();
}

int gk_edit_distance(const uint8_t* d_reads, const uint8_t* d_refs, int64_t stride,
                     int64_t n_pairs, int32_t len, int32_t* d_dist, void* stream) {
  int rc = check_ascii(d_reads, n_pairs, len, stride);
  if (rc) return rc;
  if (n_pairs == 0) return GK_OK;
  if (!d_refs || !d_dist) return GK_ERR_ARG;
  if (!aligned(d_dist, 4)) return GK_ERR_ALIGN;
  gk::launch_edit_distance(d_reads, d_refs, stride, n_pairs, len, d_dist, (cudaStream_t)stream);
  return after_launch();
}

int gk_accuracy(const uint32_t* d_accept_bits, int64_t bits_row_stride, const uint8_t* d_errcount,
                int64_t err_row_stride, const int32_t* d_dist, int64_t n_pairs,
                const int32_t* d_e_list, int32_t n_rows, uint64_t* d_counts, void* stream) {
  if (n_pairs < 0 || n_rows < 0 || n_rows > 65535) return GK_ERR_ARG;
  if (n_rows == 0) return GK_OK;
  if (!d_counts || !d_e_list) return GK_ERR_ARG;
  if (!aligned(d_counts, 8) || !aligned(d_e_list, 4)) return GK_ERR_ALIGN;
  if (n_pairs == 0)
    return cuda_status(cudaMemsetAsync(d_counts, 0, 32 * (size_t)n_rows, (cudaStream_t)stream));
  if (!d_accept_bits || !d_errcount || !d_dist) return GK_ERR_ARG;
  if (n_rows > 1 && (bits_row_stride < (int64_t)gk_result_words(n_pairs) ||
                     err_row_stride < n_pairs))
    return GK_ERR_ARG;
  if (!aligned(d_accept_bits, 4) || !aligned(d_dist, 4)) return GK_ERR_ALIGN;
  gk::launch_accuracy(d_accept_bits, bits_row_stride, d_errcount, err_row_stride, d_dist, n_pairs,
                      d_e_list, n_rows, reinterpret_cast<unsigned long long*>(d_counts),
                      (cudaStream_t)stream);
  return after_launch();
}

// ---- host-buffer end-to-end pipelines -----------------------------------------
// Chunks of pairs stream through two buffer sets on two CUDA streams, so the
// host->device copy of chunk c+1 overlaps the kernels of chunk c and the
// device->host copy of chunk c-1 (the paper's "filter time").
// The streams, events and a small pinned count buffer are created once per
// (host thread, device) and reused across calls.  Every call is ordered after
// the work already enqueued on the caller's `stream` (its internal streams wait
// on an event recorded there) and returns once the results are in host memory.
static size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

namespace {
struct HostRes {
  bool ready = false;
  cudaStream_t st[2];
  cudaEvent_t ev_in, ev_cnt[2];
  unsigned long long* cnt = nullptr;  // pinned, 2 counts
};
constexpr int kMaxDev = 64;
thread_local HostRes g_host[kMaxDev];

int host_begin(void* stream, HostRes** out) {
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return cuda_status(err);
  if (dev < 0 || dev >= kMaxDev) return GK_ERR_ARG;
  HostRes& r = g_host[dev];
  if (!r.ready) {
    // create everything or nothing: a partial failure releases what was created
    HostRes t;
    t.st[0] = t.st[1] = nullptr;
    t.ev_in = t.ev_cnt[0] = t.ev_cnt[1] = nullptr;
    for (int b = 0; b < 2 && err == cudaSuccess; ++b) {
      err = cudaStreamCreateWithFlags(&t.st[b], cudaStreamNonBlocking);
      if (err == cudaSuccess) err = cudaEventCreateWithFlags(&t.ev_cnt[b], cudaEventDisableTiming);
    }
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&t.ev_in, cudaEventDisableTiming);
    if (err == cudaSuccess)
      err = cudaHostAlloc(reinterpret_cast<void**>(&t.cnt), 2 * sizeof(unsigned long long),
                          cudaHostAllocDefault);
    if (err != cudaSuccess) {
      for (int b = 0; b < 2; ++b) {
        if (t.st[b]) cudaStreamDestroy(t.st[b]);
        if (t.ev_cnt[b]) cudaEventDestroy(t.ev_cnt[b]);
      }
      if (t.ev_in) cudaEventDestroy(t.ev_in);
      return cuda_status(err);
    }
    t.ready = true;
    r = t;
  }
  // order both pipeline streams after the caller's stream (its producers of
  // device inputs / workspace)
  if ((err = cudaEventRecord(r.ev_in, (cudaStream_t)stream)) != cudaSuccess) return cuda_status(err);
  for (int b = 0; b < 2; ++b)
    if ((err = cudaStreamWaitEvent(r.st[b], r.ev_in, 0)) != cudaSuccess) return cuda_status(err);
  *out = &r;
  return GK_OK;
}

int host_end(HostRes* r, int rc) {
  for (int b = 0; b < 2; ++b) {
    cudaError_t err = cudaStreamSynchronize(r->st[b]);
    if (rc == GK_OK && err != cudaSuccess) rc = cuda_status(err);
  }
  return rc;
}

// Index lists of a chunked pipeline: chunk c's accepted indices (absolute, written
// by the compaction kernel with base p0) are copied back once its count is known
// -- the host waits for chunk c-1's count while chunk c runs.
struct IdxDrain {
  HostRes* r;
  uint32_t* h_idx;
  unsigned long long total = 0;
  int pending = -1;         // buffer set of the chunk waiting to be drained
  const uint32_t* d_idx[2];
  int drain() {
    if (pending < 0) return GK_OK;
    const int b = pending;
    pending = -1;
    cudaError_t err = cudaEventSynchronize(r->ev_cnt[b]);
    if (err != cudaSuccess) return cuda_status(err);
    const unsigned long long n = r->cnt[b];
    if (n) {
      err = cudaMemcpyAsync(h_idx + total, d_idx[b], (size_t)n * 4, cudaMemcpyDeviceToHost,
                            r->st[b]);
      if (err != cudaSuccess) return cuda_status(err);
    }
    total += n;
    return GK_OK;
  }
};
}  // namespace

struct HostLayout {
  size_t in, packed, undef, acc, err, idx, nacc, cws, per_set;
};

static HostLayout host_layout(int64_t chunk, int64_t stride, int32_t len, int32_t rows) {
  HostLayout L;
  L.in = round_up((size_t)chunk * (size_t)stride, 256);
  L.packed = round_up(gk_packed_words(chunk, len) * 4, 256);
  L.undef = round_up(gk_undef_words(chunk) * 4, 256);
  L.acc = round_up((size_t)(chunk / 32) * 4, 256);  // chunk is a multiple of 1024
  L.err = round_up((size_t)chunk, 256);
  L.idx = round_up((size_t)chunk * 4, 256);
  L.nacc = 256;
  L.cws = round_up(gk::compact_workspace_bytes(chunk), 256);
  L.per_set = 2 * L.in + 2 * L.packed + 2 * L.undef + (size_t)rows * (L.acc + L.err) + L.idx +
              L.nacc + L.cws;
  return L;
}

struct SetPtrs {
  uint8_t *r, *f;
  uint32_t *pq, *pr, *uq, *ur, *acc;
  uint8_t* err;
  uint32_t* idx;
  uint64_t* nacc;
  void* cws;
};

static SetPtrs set_ptrs(void* ws, const HostLayout& L, int b, int rows) {
  uint8_t* p = static_cast<uint8_t*>(ws) + (size_t)b * L.per_set;
  SetPtrs s;
  s.r = p; p += L.in;
  s.f = p; p += L.in;
  s.pq = reinterpret_cast<uint32_t*>(p); p += L.packed;
  s.pr = reinterpret_cast<uint32_t*>(p); p += L.packed;
  s.uq = reinterpret_cast<uint32_t*>(p); p += L.undef;
  s.ur = reinterpret_cast<uint32_t*>(p); p += L.undef;
  s.acc = reinterpret_cast<uint32_t*>(p); p += (size_t)rows * L.acc;
  s.err = p; p += (size_t)rows * L.err;
  s.idx = reinterpret_cast<uint32_t*>(p); p += L.idx;
  s.nacc = reinterpret_cast<uint64_t*>(p); p += L.nacc;
  s.cws = p;
  return s;
}

size_t gk_host_workspace_bytes(int64_t chunk_pairs, int64_t stride, int32_t len) {
  if (chunk_pairs <= 0 || stride <= 0 || len <= 0) return 0;
  return 2 * host_layout(chunk_pairs, stride, len, 1).per_set;
}

int gk_filter_host(const uint8_t* h_reads, const uint8_t* h_refs, int64_t stride,
                   int64_t n_pairs, int32_t len, int32_t e, uint32_t* h_accept_bits,
                   uint8_t* h_errcount, uint32_t* h_idx, uint64_t* h_n_acc, void* d_ws,
                   size_t ws_bytes, int64_t chunk_pairs, void* stream) {
  int rc = check_ascii(h_reads, n_pairs, len, stride);
  if (rc) return rc;
  if (e < 0 || e >= len) return GK_ERR_E;
  if (h_idx && !h_n_acc) return GK_ERR_ARG;
  if (h_idx && n_pairs >= ((int64_t)1 << 32)) return GK_ERR_ARG;
  if (n_pairs == 0) {
    if (h_n_acc) *h_n_acc = 0;
    return GK_OK;
  }
  if (!h_refs || (!h_accept_bits && !h_idx)) return GK_ERR_ARG;
  if (chunk_pairs <= 0 || chunk_pairs % 1024 != 0) return GK_ERR_ARG;
  if (!d_ws || ws_bytes < gk_host_workspace_bytes(chunk_pairs, stride, len))
    return GK_ERR_WORKSPACE;
  if (!aligned(d_ws, 256)) return GK_ERR_ALIGN;
  const HostLayout L = host_layout(chunk_pairs, stride, len, 1);
  HostRes* res = nullptr;
  if ((rc = host_begin(stream, &res)) != GK_OK) return rc;
  IdxDrain drain{res, h_idx};
  const int64_t nchunks = (n_pairs + chunk_pairs - 1) / chunk_pairs;
  for (int64_t c = 0; c < nchunks && rc == GK_OK; ++c) {
    const int b = (int)(c & 1);
    cudaStream_t st = res->st[b];
    const SetPtrs s = set_ptrs(d_ws, L, b, 1);
    drain.d_idx[b] = s.idx;
    const int64_t p0 = c * chunk_pairs;
    const int64_t np = (n_pairs - p0) < chunk_pairs ? (n_pairs - p0) : chunk_pairs;
    const size_t bytes = (size_t)((np - 1) * stride + len);
    cudaError_t err = cudaMemcpyAsync(s.r, h_reads + p0 * stride, bytes, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(s.f, h_refs + p0 * stride, bytes, cudaMemcpyHostToDevice, st);
    if (err != cudaSuccess) { rc = cuda_status(err); break; }
    // a1 twice, a2-a6 (the same kernels as gk_encode + gk_filter), a7 if asked
    gk::launch_encode(s.r, np, len, stride, s.pq, s.uq, st);
    gk::launch_encode(s.f, np, len, stride, s.pr, s.ur, st);
    gk::launch_filter(s.pq, s.pr, s.uq, s.ur, np, len, e, s.acc, h_errcount ? s.err : nullptr, 0, st);
    if (h_idx)
      gk::launch_compact(s.acc, np, s.idx, s.nacc, s.cws, st, 1, 0, 0, (uint32_t)p0);
    if ((rc = after_launch()) != GK_OK) break;
    if (h_accept_bits)
      err = cudaMemcpyAsync(h_accept_bits + p0 / 32, s.acc, (size_t)((np + 31) / 32) * 4,
                            cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess && h_errcount)
      err = cudaMemcpyAsync(h_errcount + p0, s.err, (size_t)np, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess && h_idx) {
      err = cudaMemcpyAsync(&res->cnt[b], s.nacc, 8, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess) err = cudaEventRecord(res->ev_cnt[b], st);
    }
    if (err != cudaSuccess) { rc = cuda_status(err); break; }
    if (h_idx) {
      if ((rc = drain.drain()) != GK_OK) break;  // chunk c-1, while chunk c runs
      drain.pending = b;
    }
  }
  if (rc == GK_OK && h_idx) rc = drain.drain();
  rc = host_end(res, rc);
  if (rc == GK_OK && h_n_acc) *h_n_acc = drain.total;
  return rc;
}

// ---- host-buffer threshold sweep ---------------------------------------------
size_t gk_host_sweep_workspace_bytes(int64_t chunk_pairs, int64_t stride, int32_t len,
                                     int32_t e_max) {
  if (chunk_pairs <= 0 || stride <= 0 || len <= 0 || e_max < 0) return 0;
  return 2 * host_layout(chunk_pairs, stride, len, e_max + 1).per_set;
}

int gk_filter_host_sweep(const uint8_t* h_reads, const uint8_t* h_refs, int64_t stride,
                         int64_t n_pairs, int32_t len, const int32_t* e_list, int32_t n_e,
                         uint32_t* h_accept_bits, uint8_t* h_errcount, void* d_ws,
                         size_t ws_bytes, int64_t chunk_pairs, void* stream) {
  int rc = check_ascii(h_reads, n_pairs, len, stride);
  if (rc) return rc;
  if (n_e <= 0 || !e_list) return GK_ERR_ARG;
  for (int t = 0; t < n_e; ++t)
    if (e_list[t] < 0 || e_list[t] >= len) return GK_ERR_E;
  if (n_pairs == 0) return GK_OK;
  if (!h_refs || !h_accept_bits) return GK_ERR_ARG;
  if (chunk_pairs <= 0 || chunk_pairs % 1024 != 0) return GK_ERR_ARG;
  int32_t e_max = 0;
  for (int t = 0; t < n_e; ++t) e_max = e_list[t] > e_max ? e_list[t] : e_max;
  if (!d_ws || ws_bytes < gk_host_sweep_workspace_bytes(chunk_pairs, stride, len, e_max))
    return GK_ERR_WORKSPACE;
  if (!aligned(d_ws, 256)) return GK_ERR_ALIGN;
  const HostLayout L = host_layout(chunk_pairs, stride, len, e_max + 1);
  const size_t words_total = gk_result_words(n_pairs);
  HostRes* res = nullptr;
  if ((rc = host_begin(stream, &res)) != GK_OK) return rc;
  const int64_t nchunks = (n_pairs + chunk_pairs - 1) / chunk_pairs;
  for (int64_t c = 0; c < nchunks && rc == GK_OK; ++c) {
    const int b = (int)(c & 1);
    cudaStream_t st = res->st[b];
    const SetPtrs s = set_ptrs(d_ws, L, b, e_max + 1);
    const int64_t p0 = c * chunk_pairs;
    const int64_t np = (n_pairs - p0) < chunk_pairs ? (n_pairs - p0) : chunk_pairs;
    const size_t bytes = (size_t)((np - 1) * stride + len);
    cudaError_t err = cudaMemcpyAsync(s.r, h_reads + p0 * stride, bytes, cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(s.f, h_refs + p0 * stride, bytes, cudaMemcpyHostToDevice, st);
    if (err != cudaSuccess) { rc = cuda_status(err); break; }
    gk::launch_encode(s.r, np, len, stride, s.pq, s.uq, st);
    gk::launch_encode(s.f, np, len, stride, s.pr, s.ur, st);
    // every e <= e_max in one pass (gk_filter_sweep); rows of the chunk: [e][np/32]
    // bits, then [e][np] counts
    uint8_t* ec = h_errcount ? s.err : nullptr;
    gk::launch_filter_sweep(s.pq, s.pr, s.uq, s.ur, np, len, e_max, s.acc, ec, 0, st);
    rc = after_launch();
    const size_t words = (size_t)((np + 31) / 32);
    for (int t = 0; t < n_e && rc == GK_OK; ++t) {
      const int e = e_list[t];
      err = cudaMemcpyAsync(h_accept_bits + (size_t)t * words_total + p0 / 32,
                            s.acc + (size_t)e * words, words * 4, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess && h_errcount)
        err = cudaMemcpyAsync(h_errcount + (size_t)t * n_pairs + p0, s.err + (size_t)e * np,
                              (size_t)np, cudaMemcpyDeviceToHost, st);
      if (err != cudaSuccess) rc = cuda_status(err);
    }
  }
  return host_end(res, rc);
}

// ---- host-buffer index mode ----------------------------------------------------
static size_t index_chunk_bytes(int64_t chunk, int32_t len, int32_t e_max) {
  const size_t offs = round_up((size_t)chunk * 16, 256);
  const size_t packed = round_up(gk_packed_words(chunk, len) * 4, 256);
  const size_t undef = round_up(gk_undef_words(chunk) * 4, 256);
  const size_t acc = round_up((size_t)(chunk / 32) * 4, 256);
  const size_t err = round_up((size_t)chunk, 256);
  return offs + 2 * packed + 2 * undef + (size_t)(e_max + 1) * (acc + err);
}

size_t gk_host_index_workspace_bytes(int64_t chunk_pairs, int32_t len, int32_t e_max) {
  if (chunk_pairs <= 0 || len <= 0 || e_max < 0) return 0;
  return 2 * index_chunk_bytes(chunk_pairs, len, e_max);
}

int gk_filter_host_index(const uint32_t* d_read_planes, int64_t read_bases,
                         const uint32_t* d_ref_planes, int64_t ref_bases,
                         const int64_t* h_read_offsets, const int64_t* h_ref_offsets,
                         int64_t n_pairs, int32_t len, int32_t e_max, uint32_t* h_accept_bits,
                         uint8_t* h_errcount, void* d_ws, size_t ws_bytes, int64_t chunk_pairs,
                         void* stream) {
  if (n_pairs < 0 || read_bases < 0 || ref_bases < 0) return GK_ERR_ARG;
  if (len < 1 || len > GK_MAX_LEN) return GK_ERR_LEN;
  if (e_max < 0 || e_max >= len) return GK_ERR_E;
  if (n_pairs == 0) return GK_OK;
  if (!d_read_planes || !d_ref_planes || !h_read_offsets || !h_ref_offsets || !h_accept_bits)
    return GK_ERR_ARG;
  if (chunk_pairs <= 0 || chunk_pairs % 1024 != 0) return GK_ERR_ARG;
  if (!d_ws || ws_bytes < gk_host_index_workspace_bytes(chunk_pairs, len, e_max))
    return GK_ERR_WORKSPACE;
  if (!aligned(d_ws, 256) || !aligned(d_read_planes, 16) || !aligned(d_ref_planes, 16))
    return GK_ERR_ALIGN;
  const size_t per_set = index_chunk_bytes(chunk_pairs, len, e_max);
  const size_t words_total = gk_result_words(n_pairs);
  const size_t acc_row = round_up((size_t)(chunk_pairs / 32) * 4, 256);
  HostRes* res = nullptr;
  int rc = host_begin(stream, &res);
  if (rc != GK_OK) return rc;
  const int64_t nchunks = (n_pairs + chunk_pairs - 1) / chunk_pairs;
  for (int64_t c = 0; c < nchunks && rc == GK_OK; ++c) {
    const int b = (int)(c & 1);
    cudaStream_t st = res->st[b];
    uint8_t* base = static_cast<uint8_t*>(d_ws) + b * per_set;
    int64_t* d_roff = reinterpret_cast<int64_t*>(base);
    int64_t* d_foff = d_roff + chunk_pairs;
    uint32_t* pq = reinterpret_cast<uint32_t*>(base + round_up((size_t)chunk_pairs * 16, 256));
    uint32_t* pr = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(pq) +
                                               round_up(gk_packed_words(chunk_pairs, len) * 4, 256));
    uint32_t* uq = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(pr) +
                                               round_up(gk_packed_words(chunk_pairs, len) * 4, 256));
    uint32_t* ur = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(uq) +
                                               round_up(gk_undef_words(chunk_pairs) * 4, 256));
    uint8_t* outs = reinterpret_cast<uint8_t*>(ur) + round_up(gk_undef_words(chunk_pairs) * 4, 256);
    const int64_t p0 = c * chunk_pairs;
    const int64_t np = (n_pairs - p0) < chunk_pairs ? (n_pairs - p0) : chunk_pairs;
    cudaError_t err = cudaMemcpyAsync(d_roff, h_read_offsets + p0, (size_t)np * 8,
                                      cudaMemcpyHostToDevice, st);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(d_foff, h_ref_offsets + p0, (size_t)np * 8, cudaMemcpyHostToDevice, st);
    if (err != cudaSuccess) { rc = cuda_status(err); break; }
    gk::launch_gather_windows(d_read_planes, read_bases, d_roff, np, len, pq, uq, st);
    gk::launch_gather_windows(d_ref_planes, ref_bases, d_foff, np, len, pr, ur, st);
    const size_t words = (size_t)((np + 31) / 32);
    uint32_t* acc = reinterpret_cast<uint32_t*>(outs);
    uint8_t* ec = h_errcount ? outs + (size_t)(e_max + 1) * acc_row : nullptr;
    gk::launch_filter_sweep(pq, pr, uq, ur, np, len, e_max, acc, ec, 0, st);
    rc = after_launch();
    for (int e = 0; e <= e_max && rc == GK_OK; ++e) {
      err = cudaMemcpyAsync(h_accept_bits + (size_t)e * words_total + p0 / 32, acc + (size_t)e * words,
                            words * 4, cudaMemcpyDeviceToHost, st);
      if (err == cudaSuccess && h_errcount)
        err = cudaMemcpyAsync(h_errcount + (size_t)e * n_pairs + p0, ec + (size_t)e * np, (size_t)np,
                              cudaMemcpyDeviceToHost, st);
      if (err != cudaSuccess) rc = cuda_status(err);
    }
  }
  return host_end(res, rc);
}

}  // extern "C"
