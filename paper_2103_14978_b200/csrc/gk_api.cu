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
int launch_pack_planes(const uint8_t* rows, int64_t n_rows, int len, int64_t stride,
                       uint32_t* planes, cudaStream_t stream);
int launch_gather_windows(const uint32_t* planes, int64_t nbases, const int64_t* offsets, int64_t n,
                          int len, uint32_t* packed, uint32_t* undef, cudaStream_t stream);
}  // namespace gk

static thread_local int g_last_cuda_error = 0;
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

int gk_pack_planes(const uint8_t* d_rows, int64_t n_rows, int32_t len, int64_t stride,
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

// ---- host-buffer end-to-end pipeline ------------------------------------------
static size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t gk_host_workspace_bytes(int64_t chunk_pairs, int64_t stride) {
  if (chunk_pairs <= 0 || stride <= 0) return 0;
  const size_t in = round_up((size_t)chunk_pairs * (size_t)stride, 256);
  const size_t acc = round_up((size_t)(chunk_pairs / 32 + 1) * 4, 256);
  const size_t err = round_up((size_t)chunk_pairs, 256);
  return 2 * (2 * in + acc + err);
}

int gk_filter_host(const uint8_t* h_reads, const uint8_t* h_refs, int64_t stride,
                   int64_t n_pairs, int32_t len, int32_t e, uint32_t* h_accept_bits,
                   uint8_t* h_errcount, void* d_ws, size_t ws_bytes, int64_t chunk_pairs) {
  int rc = check_ascii(h_reads, n_pairs, len, stride);
  if (rc) return rc;
  if (e < 0 || e >= len) return GK_ERR_E;
  if (n_pairs == 0) return GK_OK;
  if (!h_refs || !h_accept_bits) return GK_ERR_ARG;
  if (chunk_pairs <= 0 || chunk_pairs % 1024 != 0) return GK_ERR_ARG;
  if (!d_ws || ws_bytes < gk_host_workspace_bytes(chunk_pairs, stride)) return GK_ERR_WORKSPACE;
  if (!aligned(d_ws, 256)) return GK_ERR_ALIGN;

  const size_t in = round_up((size_t)chunk_pairs * (size_t)stride, 256);
  const size_t acc = round_up((size_t)(chunk_pairs / 32 + 1) * 4, 256);
  const size_t errb = round_up((size_t)chunk_pairs, 256);
  uint8_t* base = static_cast<uint8_t*>(d_ws);
  struct Buf { uint8_t *r, *f; uint32_t* a; uint8_t* c; } buf[2];
  for (int b = 0; b < 2; ++b) {
    uint8_t* p = base + b * (2 * in + acc + errb);
    buf[b].r = p;
    buf[b].f = p + in;
    buf[b].a = reinterpret_cast<uint32_t*>(p + 2 * in);
    buf[b].c = p + 2 * in + acc;
  }
  cudaStream_t st[2];
  for (int b = 0; b < 2; ++b) {
    cudaError_t err = cudaStreamCreateWithFlags(&st[b], cudaStreamNonBlocking);
    if (err != cudaSuccess) {
      if (b == 1) cudaStreamDestroy(st[0]);
      return cuda_status(err);
    }
  }
  rc = GK_OK;
  const int64_t nchunks = (n_pairs + chunk_pairs - 1) / chunk_pairs;
  for (int64_t c = 0; c < nchunks && rc == GK_OK; ++c) {
    const int b = (int)(c & 1);
    const int64_t p0 = c * chunk_pairs;
    const int64_t np = (n_pairs - p0) < chunk_pairs ? (n_pairs - p0) : chunk_pairs;
    const size_t bytes = (size_t)((np - 1) * stride + len);
    cudaError_t err = cudaMemcpyAsync(buf[b].r, h_reads + p0 * stride, bytes,
                                      cudaMemcpyHostToDevice, st[b]);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(buf[b].f, h_refs + p0 * stride, bytes, cudaMemcpyHostToDevice, st[b]);
    if (err != cudaSuccess) { rc = cuda_status(err); break; }
    gk::launch_filter_ascii(buf[b].r, buf[b].f, stride, np, len, e, buf[b].a,
                            h_errcount ? buf[b].c : nullptr, st[b]);
    rc = after_launch();
    if (rc) break;
    err = cudaMemcpyAsync(h_accept_bits + p0 / 32, buf[b].a, (size_t)((np + 31) / 32) * 4,
                          cudaMemcpyDeviceToHost, st[b]);
    if (err == cudaSuccess && h_errcount)
      err = cudaMemcpyAsync(h_errcount + p0, buf[b].c, (size_t)np, cudaMemcpyDeviceToHost, st[b]);
    if (err != cudaSuccess) { rc = cuda_status(err); break; }
  }
  for (int b = 0; b < 2; ++b) {
    cudaError_t err = cudaStreamSynchronize(st[b]);
    if (rc == GK_OK && err != cudaSuccess) rc = cuda_status(err);
    cudaStreamDestroy(st[b]);
  }
  return rc;
}

// ---- host-buffer threshold sweep ---------------------------------------------
struct SweepLayout {
  size_t in, packed, undef, acc, err, per_set;
};

static SweepLayout sweep_layout(int64_t chunk, int64_t stride, int32_t len, int32_t e_max) {
  SweepLayout L;
  L.in = round_up((size_t)chunk * (size_t)stride, 256);
  L.packed = round_up(gk_packed_words(chunk, len) * 4, 256);
  L.undef = round_up(gk_undef_words(chunk) * 4, 256);
  L.acc = round_up((size_t)(chunk / 32) * 4, 256);  // chunk is a multiple of 1024
  L.err = round_up((size_t)chunk, 256);
  L.per_set = 2 * L.in + 2 * L.packed + 2 * L.undef + (size_t)(e_max + 1) * (L.acc + L.err);
  return L;
}

size_t gk_host_sweep_workspace_bytes(int64_t chunk_pairs, int64_t stride, int32_t len,
                                     int32_t e_max) {
  if (chunk_pairs <= 0 || stride <= 0 || len <= 0 || e_max < 0) return 0;
  return 2 * sweep_layout(chunk_pairs, stride, len, e_max).per_set;
}

int gk_filter_host_sweep(const uint8_t* h_reads, const uint8_t* h_refs, int64_t stride,
                         int64_t n_pairs, int32_t len, const int32_t* e_list, int32_t n_e,
                         uint32_t* h_accept_bits, uint8_t* h_errcount, void* d_ws,
                         size_t ws_bytes, int64_t chunk_pairs) {
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
  const SweepLayout L = sweep_layout(chunk_pairs, stride, len, e_max);
  const size_t words_total = gk_result_words(n_pairs);
  cudaStream_t st[2];
  for (int b = 0; b < 2; ++b) {
    cudaError_t err = cudaStreamCreateWithFlags(&st[b], cudaStreamNonBlocking);
    if (err != cudaSuccess) {
      if (b == 1) cudaStreamDestroy(st[0]);
      return cuda_status(err);
    }
  }
  rc = GK_OK;
  const int64_t nchunks = (n_pairs + chunk_pairs - 1) / chunk_pairs;
  for (int64_t c = 0; c < nchunks && rc == GK_OK; ++c) {
    const int b = (int)(c & 1);
    uint8_t* base = static_cast<uint8_t*>(d_ws) + b * L.per_set;
    uint8_t* dr = base;
    uint8_t* df = dr + L.in;
    uint32_t* pq = reinterpret_cast<uint32_t*>(df + L.in);
    uint32_t* pr = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(pq) + L.packed);
    uint32_t* uq = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(pr) + L.packed);
    uint32_t* ur = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(uq) + L.undef);
    uint8_t* outs = reinterpret_cast<uint8_t*>(ur) + L.undef;
    const int64_t p0 = c * chunk_pairs;
    const int64_t np = (n_pairs - p0) < chunk_pairs ? (n_pairs - p0) : chunk_pairs;
    const size_t bytes = (size_t)((np - 1) * stride + len);
    cudaError_t err = cudaMemcpyAsync(dr, h_reads + p0 * stride, bytes, cudaMemcpyHostToDevice,
                                      st[b]);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(df, h_refs + p0 * stride, bytes, cudaMemcpyHostToDevice, st[b]);
    if (err != cudaSuccess) { rc = cuda_status(err); break; }
    gk::launch_encode(dr, np, len, stride, pq, uq, st[b]);
    gk::launch_encode(df, np, len, stride, pr, ur, st[b]);
    // every e <= e_max in one pass (gk_filter_sweep); rows of the chunk: [e][chunk/32] bits,
    // then [e][chunk] counts
    uint32_t* acc = reinterpret_cast<uint32_t*>(outs);
    uint8_t* ec = h_errcount ? outs + (size_t)(e_max + 1) * L.acc : nullptr;
    gk::launch_filter_sweep(pq, pr, uq, ur, np, len, e_max, acc, ec, 0, st[b]);
    rc = after_launch();
    const size_t words = (size_t)((np + 31) / 32);
    for (int t = 0; t < n_e && rc == GK_OK; ++t) {
      const int e = e_list[t];
      err = cudaMemcpyAsync(h_accept_bits + (size_t)t * words_total + p0 / 32,
                            acc + (size_t)e * words, words * 4, cudaMemcpyDeviceToHost, st[b]);
      if (err == cudaSuccess && h_errcount)
        err = cudaMemcpyAsync(h_errcount + (size_t)t * n_pairs + p0, ec + (size_t)e * np,
                              (size_t)np, cudaMemcpyDeviceToHost, st[b]);
      if (err != cudaSuccess) rc = cuda_status(err);
    }
  }
  for (int b = 0; b < 2; ++b) {
    cudaError_t err = cudaStreamSynchronize(st[b]);
    if (rc == GK_OK && err != cudaSuccess) rc = cuda_status(err);
    cudaStreamDestroy(st[b]);
  }
  return rc;
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
                         uint8_t* h_errcount, void* d_ws, size_t ws_bytes, int64_t chunk_pairs) {
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
  cudaStream_t st[2];
  for (int b = 0; b < 2; ++b) {
    cudaError_t err = cudaStreamCreateWithFlags(&st[b], cudaStreamNonBlocking);
    if (err != cudaSuccess) {
      if (b == 1) cudaStreamDestroy(st[0]);
      return cuda_status(err);
    }
  }
  int rc = GK_OK;
  const int64_t nchunks = (n_pairs + chunk_pairs - 1) / chunk_pairs;
  for (int64_t c = 0; c < nchunks && rc == GK_OK; ++c) {
    const int b = (int)(c & 1);
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
                                      cudaMemcpyHostToDevice, st[b]);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(d_foff, h_ref_offsets + p0, (size_t)np * 8, cudaMemcpyHostToDevice,
                            st[b]);
    if (err != cudaSuccess) { rc = cuda_status(err); break; }
    gk::launch_gather_windows(d_read_planes, read_bases, d_roff, np, len, pq, uq, st[b]);
    gk::launch_gather_windows(d_ref_planes, ref_bases, d_foff, np, len, pr, ur, st[b]);
    const size_t words = (size_t)((np + 31) / 32);
    uint32_t* acc = reinterpret_cast<uint32_t*>(outs);
    uint8_t* ec = h_errcount ? outs + (size_t)(e_max + 1) * round_up((size_t)(chunk_pairs / 32) * 4, 256)
                             : nullptr;
    gk::launch_filter_sweep(pq, pr, uq, ur, np, len, e_max, acc, ec, 0, st[b]);
    rc = after_launch();
    for (int e = 0; e <= e_max && rc == GK_OK; ++e) {
      err = cudaMemcpyAsync(h_accept_bits + (size_t)e * words_total + p0 / 32, acc + (size_t)e * words,
                            words * 4, cudaMemcpyDeviceToHost, st[b]);
      if (err == cudaSuccess && h_errcount)
        err = cudaMemcpyAsync(h_errcount + (size_t)e * n_pairs + p0, ec + (size_t)e * np, (size_t)np,
                              cudaMemcpyDeviceToHost, st[b]);
      if (err != cudaSuccess) rc = cuda_status(err);
    }
  }
  for (int b = 0; b < 2; ++b) {
    cudaError_t err = cudaStreamSynchronize(st[b]);
    if (rc == GK_OK && err != cudaSuccess) rc = cuda_status(err);
    cudaStreamDestroy(st[b]);
  }
  return rc;
}

}  // extern "C"
