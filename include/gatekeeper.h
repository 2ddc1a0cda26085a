/* gatekeeper.h -- C ABI of the B200-native GateKeeper-GPU pre-alignment filter.
 *
 * Method: Bingol et al., "GateKeeper-GPU: Fast and Accurate Pre-Alignment
 * Filtering in Short Read Mapping", arXiv 2103.14978.  For every
 * (read, candidate reference segment) pair of equal length L and an edit
 * threshold e the filter (Fig. S.1 :444-490):
 *   1. 2-bit encodes both sequences (A=00 C=01 G=10 T=11, :49);
 *   2. passes pairs containing a non-ACGT byte unfiltered (:95);
 *   3. builds the Hamming mask, amends it and counts its errors; a count <= e
 *      accepts immediately (Fig. S.1 "e > E, therefore ASM begins", :466);
 *   4. otherwise builds 2e shifted masks (read shifted k = 1..e bases toward
 *      higher / lower positions), amends every mask (turns bounded 0-runs of
 *      length <= 2 into 1s, :51), forces the vacated leading / trailing bits
 *      to 1 (GateKeeper-GPU's edge fix, :109), ANDs all 2e+1 masks (:51);
 *   5. counts errors in 4-base windows (runs of 1s per window, :51) and
 *      rejects iff the count exceeds e (:51); reports the count (:166).
 * The exact readings of the passages the paper leaves open are listed in
 * DESIGN.md ("Readings of the paper", R1-R13).
 *
 * Conventions (all entry points):
 *  - Every pointer named d_* is a DEVICE pointer (e.g. torch.Tensor.data_ptr()
 *    of a CUDA tensor); h_* is a HOST pointer.  The caller owns every buffer;
 *    the library never allocates, frees or retains a pointer past the call.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Device calls are asynchronous and ordered on `stream`.
 *  - Arguments are validated on the host before any launch.  Return value:
 *    GK_OK (0) or a negative gk_status.  A launch failure returns GK_ERR_CUDA;
 *    gk_last_cuda_error() then gives the cudaError_t (thread-local).
 *  - n = 0 is a valid no-op.  1 <= len <= GK_MAX_LEN; 0 <= e < len.
 *  - No global mutable state (apart from the diagnostic launch counter of
 *    gk_launch_count, an atomic); calls from several host threads are safe.
 *
 * Packed sequence layout ("bit-sliced tiles", written by gk_encode, read by
 * gk_filter).  Sequences are grouped by 32 ("group") and groups by 32
 * ("tile" = 1024 sequences).  Sequence s lives in tile t = s/1024, lane
 * g = (s/32)%32, bit j = s%32.  For base i (0 <= i < len) the two 32-bit words
 *     d_packed[((t*len + i)*32 + g)*2 + 0]   plane 0 = high bit of the code
 *     d_packed[((t*len + i)*32 + g)*2 + 1]   plane 1 = low  bit of the code
 * hold, at bit j, that bit of sequence s's base i.  So one 32-bit word carries
 * one base position of 32 sequences, and a warp reading position i of a tile
 * reads 256 contiguous bytes.  Total size: gk_packed_words(n, len) words
 * (= ceil(n/1024)*len*64, i.e. len/4 bytes per sequence).  Sequences
 * s >= n in the last tile are encoded as all-'A' and defined.
 * d_undef[t*32 + g] bit j = 1 iff sequence s contains a byte outside
 * {A,C,G,T,a,c,g,t} ("undefined"); the plane bits of an
 * undefined sequence are unspecified.
 *
 * Result layout.  d_accept_bits[p/32] bit p%32 = 1 iff pair p is accepted
 * ("1" = accept, "0" = reject); gk_result_words(n) words, bits of
 * pairs >= n in the last word are 0.  d_errcount[p] (optional, may be NULL) =
 * the approximate edit distance the deciding stage counted (0..254), or 255 for
 * an undefined pair.
 */
#ifndef GATEKEEPER_H
#define GATEKEEPER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GK_MAX_LEN 508      /* max count 2*ceil(508/4) = 254 fits a byte; 255 = undefined */
#define GK_MAX_STRIDE 1024  /* row stride limit of the ASCII entry points */
#define GK_TILE 1024        /* sequences per packed tile */

typedef enum gk_status {
  GK_OK = 0,
  GK_ERR_ARG = -1,       /* NULL pointer where one is required, n < 0, stride < len, ... */
  GK_ERR_LEN = -2,       /* len outside [1, GK_MAX_LEN] */
  GK_ERR_E = -3,         /* e outside [0, len) */
  GK_ERR_ALIGN = -4,     /* packed / result buffer not 4-byte (words) or 16-byte aligned */
  GK_ERR_WORKSPACE = -5, /* workspace NULL or smaller than the *_workspace_bytes() query */
  GK_ERR_CUDA = -6       /* a CUDA call failed; see gk_last_cuda_error() */
} gk_status;

/* Library version (major*10000 + minor*100 + patch). */
int gk_version(void);
/* Static, NUL-terminated description of a status code. */
const char* gk_status_string(int status);
/* cudaError_t of the last GK_ERR_CUDA returned on this host thread (0 if none). */
int gk_last_cuda_error(void);
/* Number of CUDA kernels this process has launched through the library so far
 * (process-wide atomic counter; the bench reads it around its timed region). */
uint64_t gk_launch_count(void);

/* Size queries (pure host functions, no CUDA). */
size_t gk_packed_words(int64_t n_seqs, int32_t len); /* u32 words of a packed sequence set */
size_t gk_undef_words(int64_t n_seqs);               /* u32 words of its undefined flags */
size_t gk_result_words(int64_t n_pairs);             /* u32 words of accept bits */

/* a1: ASCII -> packed bit-sliced tiles (device encoding :105).
 *  d_seqs   : n_seqs rows of `stride` bytes, base i of row s at d_seqs[s*stride+i];
 *             only the first len bytes of a row are read.  len <= stride <= GK_MAX_STRIDE.
 *  d_packed : gk_packed_words(n_seqs, len) u32, 16-byte aligned (written).
 *  d_undef  : gk_undef_words(n_seqs) u32, 4-byte aligned (written).
 * Every byte of the two outputs is written (tail sequences as all-'A').
 * Errors: GK_ERR_ARG (NULL, n_seqs < 0, stride < len or > GK_MAX_STRIDE),
 * GK_ERR_LEN, GK_ERR_ALIGN, GK_ERR_CUDA. */
int gk_encode(const uint8_t* d_seqs, int64_t n_seqs, int32_t len, int64_t stride,
              uint32_t* d_packed, uint32_t* d_undef, void* stream);

/* a2-a6: the filtration of n_pairs packed pairs (read p = sequence p of
 * d_reads_packed, reference segment p = sequence p of d_refs_packed; both sets
 * encoded by gk_encode with the same n and len).
 *  d_accept_bits : gk_result_words(n_pairs) u32 (written).
 *  d_errcount    : n_pairs bytes (written) or NULL.
 * Errors: GK_ERR_ARG, GK_ERR_LEN, GK_ERR_E, GK_ERR_ALIGN, GK_ERR_CUDA. */
int gk_filter(const uint32_t* d_reads_packed, const uint32_t* d_refs_packed,
              const uint32_t* d_read_undef, const uint32_t* d_ref_undef,
              int64_t n_pairs, int32_t len, int32_t e,
              uint32_t* d_accept_bits, uint8_t* d_errcount, void* stream);

/* gk_filter with option flags.  GK_FLAG_GENERIC forces the mask-major fallback
 * kernel (F kept in shared memory, one mask at a time; never the default --
 * diagnostic / test knob: results are identical).  GK_FLAG_NO_EDGE_FIX runs the
 * ORIGINAL GateKeeper (Alser et al. 2017; PAPER.md Fig. S.1): the vacated
 * leading / trailing bits of the shifted masks stay at their amended value 0
 * instead of being ORed to 1 -- for A/B accuracy studies
 * (:136, :238); it runs on the block-transposed kernel. */
#define GK_FLAG_GENERIC 1
#define GK_FLAG_NO_EDGE_FIX 2
/* GK_FLAG_BLOCKED forces the block-transposed kernel (16-position blocks x all
 * masks, any e; the default for e above the all-register instantiations) --
 * diagnostic / test knob: results are identical. */
#define GK_FLAG_BLOCKED 4
int gk_filter_ex(const uint32_t* d_reads_packed, const uint32_t* d_refs_packed,
                 const uint32_t* d_read_undef, const uint32_t* d_ref_undef,
                 int64_t n_pairs, int32_t len, int32_t e,
                 uint32_t* d_accept_bits, uint8_t* d_errcount, int32_t flags, void* stream);

/* a2-a6 for EVERY threshold e = 0..e_max in one pass (
 * the paper sweeps e from 0 to 10% of L).  The final bit-vector
 * of threshold e is F_e = F_{e-1} & A*D_e & A*I_e, so the
 * masks of shift k serve every e >= k and one pass over the 2*e_max+1 masks
 * yields all e_max+1 decisions.  Results are identical to e_max+1 gk_filter
 * calls (including the Hamming-stage early accept of each e, readings R5/R9).
 *  d_accept_bits : (e_max+1) rows of gk_result_words(n_pairs) u32, row e =
 *                  threshold e, bit p%32 of word p/32 (written).
 *  d_errcount    : (e_max+1) rows of n_pairs bytes, row e (written) or NULL.
 *  flags         : 0 or GK_FLAG_NO_EDGE_FIX (original GateKeeper).
 * Same inputs, alignment and ownership as gk_filter.  (Beyond ~100
 * thresholds the per-e counters no longer fit in shared memory and the rows
 * come from one gk_filter launch per e: same results, no one-pass speed-up.)
 * Errors: GK_ERR_ARG, GK_ERR_LEN, GK_ERR_E (e_max outside [0, len)),
 * GK_ERR_ALIGN, GK_ERR_CUDA. */
int gk_filter_sweep(const uint32_t* d_reads_packed, const uint32_t* d_refs_packed,
                    const uint32_t* d_read_undef, const uint32_t* d_ref_undef,
                    int64_t n_pairs, int32_t len, int32_t e_max,
                    uint32_t* d_accept_bits, uint8_t* d_errcount, int32_t flags, void* stream);

/* a1-a6 in one launch from ASCII (the paper's "device-encoded" kernel, :105):
 * same inputs as two gk_encode calls (reads and refs share `stride`), same
 * outputs as gk_filter; no packed intermediate is written to HBM.
 * Errors: as gk_encode + GK_ERR_E. */
int gk_filter_ascii(const uint8_t* d_reads, const uint8_t* d_refs, int64_t stride,
                    int64_t n_pairs, int32_t len, int32_t e,
                    uint32_t* d_accept_bits, uint8_t* d_errcount, void* stream);

/* a1-a6 for EVERY threshold e = 0..e_max in one launch from ASCII: the encode of
 * gk_filter_ascii and the one-pass sweep of gk_filter_sweep fused (one CTA per
 * tile of 1024 pairs; the 2-bit planes stay in shared memory).  Outputs as
 * gk_filter_sweep (row e = threshold e; row stride gk_result_words(n_pairs)
 * words / n_pairs bytes).
 *  d_reads, d_refs : 16-byte aligned (else GK_ERR_ALIGN).
 * Errors: as gk_filter_ascii; GK_ERR_LEN also when the tile and the per-e
 * counters do not fit in shared memory (about len * 512 + e_max * 3.5 KB bytes
 * > 227 KB, e.g. 250 bp with e_max = 25): use gk_encode + gk_filter_sweep. */
int gk_filter_ascii_sweep(const uint8_t* d_reads, const uint8_t* d_refs, int64_t stride,
                          int64_t n_pairs, int32_t len, int32_t e_max,
                          uint32_t* d_accept_bits, uint8_t* d_errcount, void* stream);

/* a7: ordered indices of the accepted pairs (the accepted
 * pairs go on to verification).
 *  d_accept_bits : as written by gk_filter for n_pairs (n_pairs < 2^32).
 *  d_idx         : room for n_pairs u32 (only the first *d_n_acc are written),
 *                  ascending pair indices.  May be NULL to only count.
 *  d_n_acc       : one u64 (written): the number of accepted pairs.
 *  d_ws          : gk_compact_workspace_bytes(n_pairs) bytes of scratch.
 * Errors: GK_ERR_ARG, GK_ERR_ALIGN, GK_ERR_WORKSPACE, GK_ERR_CUDA. */
size_t gk_compact_workspace_bytes(int64_t n_pairs);
int gk_compact(const uint32_t* d_accept_bits, int64_t n_pairs, uint32_t* d_idx,
               uint64_t* d_n_acc, void* d_ws, size_t ws_bytes, void* stream);

/* a7 for a batch of rows at once (e.g. the e_max+1 rows of gk_filter_sweep):
 * row r of accept bits at d_accept_bits + r*bits_row_stride (u32 words, >=
 * gk_result_words(n_pairs) when n_rows > 1), its indices at d_idx +
 * r*idx_row_stride (u32, >= n_pairs when n_rows > 1; d_idx may be NULL to only
 * count), its count at d_n_acc[r].  One launch pair for all rows.
 *  d_ws : gk_compact_rows_workspace_bytes(n_pairs, n_rows) bytes of scratch.
 * Errors: as gk_compact (0 <= n_rows <= 65535). */
size_t gk_compact_rows_workspace_bytes(int64_t n_pairs, int32_t n_rows);
int gk_compact_rows(const uint32_t* d_accept_bits, int32_t n_rows, int64_t bits_row_stride,
                    int64_t n_pairs, uint32_t* d_idx, int64_t idx_row_stride, uint64_t* d_n_acc,
                    void* d_ws, size_t ws_bytes, void* stream);

/* Reference-index mode (section 3.5
 * :148-152): the reference genome is encoded once into bit planes, and each
 * candidate pair takes its L-base window from them at any base offset, so
 * neither an ASCII copy of every reference segment nor a per-pair encode is
 * needed.  Reads are packed the same way (row r = bases [r*len, r*len+len)).
 *
 * Bit planes of n_bases bases: gk_plane_words(n_bases) blocks of 4 u32
 * (16 bytes, interleaved so that a window at a random offset touches 2-3
 * sectors): block w = {hi, lo, undef, 0}, bit b of each describing base
 * 32w+b: hi = high code bit, lo = low code bit (A=00 C=01 G=10 T=11,
 * PAPER.md:49), undef = 1 iff the byte is not one of A C G T a c g t (:95,
 * reading R8; its code bits are 0).  One block of look-ahead past the last
 * base is included (and zeroed).  The array must be 16-byte aligned. */
size_t gk_plane_words(int64_t n_bases);

/* ASCII rows -> bit planes: base i of row r (byte d_rows[r*stride + i], i < len)
 * is base r*len + i of the planes (n_bases = n_rows*len; a genome is one row:
 * len is 64-bit, so a whole GRCh37-sized genome, ~3.1 Gbases, fits one row).
 * Contiguous input (one row, or stride == len) at a 16-byte aligned d_rows takes
 * the coalesced 16-byte-load path; any other layout is read byte by byte.
 * Errors: GK_ERR_ARG, GK_ERR_LEN, GK_ERR_ALIGN, GK_ERR_CUDA. */
int gk_pack_planes(const uint8_t* d_rows, int64_t n_rows, int64_t len, int64_t stride,
                   uint32_t* d_planes, void* stream);

/* Windows -> the packed layout gk_filter / gk_filter_sweep consume: sequence p
 * of the output (n_pairs sequences of `len` bases, gk_packed_words(n_pairs, len)
 * words + gk_undef_words(n_pairs) undefined-flag words, as written by
 * gk_encode) is bases [d_offsets[p], d_offsets[p] + len) of the planes.  A
 * window with an undefined base -- or one reaching outside [0, n_bases) -- is
 * flagged undefined (the pair is accepted with error count 255).
 *  d_offsets : n_pairs int64 base offsets in device memory (8-byte aligned).
 * Errors: GK_ERR_ARG, GK_ERR_LEN, GK_ERR_ALIGN, GK_ERR_CUDA. */
int gk_gather_windows(const uint32_t* d_planes, int64_t n_bases, const int64_t* d_offsets,
                      int64_t n_pairs, int32_t len, uint32_t* d_packed, uint32_t* d_undef,
                      void* stream);

/* Index mode from HOST candidate lists (the mapper-facing end-to-end call):
 * the read and genome planes are resident on the device (gk_pack_planes);
 * per chunk only the two int64 offsets of each pair cross PCIe (16 bytes per
 * pair instead of 2*len ASCII bytes), are gathered into the packed layout and
 * filtered for every e <= e_max in one sweep pass; the result rows come back.
 *  h_read_offsets, h_ref_offsets : n_pairs int64 base offsets (host memory;
 *                                  pinned for full PCIe bandwidth).
 *  h_accept_bits : (e_max+1) rows of gk_result_words(n_pairs) u32 (host, written).
 *  h_errcount    : (e_max+1) rows of n_pairs bytes (host, written) or NULL.
 *  d_ws          : gk_host_index_workspace_bytes(chunk_pairs, len, e_max) bytes,
 *                  256-byte aligned; chunk_pairs a multiple of 1024.
 *  stream        : the call is ordered after all work already enqueued on it (e.g.
 *                  the gk_pack_planes that produced the planes); see gk_filter_host.
 * Synchronous.  Errors: as gk_gather_windows + GK_ERR_E, GK_ERR_WORKSPACE. */
size_t gk_host_index_workspace_bytes(int64_t chunk_pairs, int32_t len, int32_t e_max);
int gk_filter_host_index(const uint32_t* d_read_planes, int64_t read_bases,
                         const uint32_t* d_ref_planes, int64_t ref_bases,
                         const int64_t* h_read_offsets, const int64_t* h_ref_offsets,
                         int64_t n_pairs, int32_t len, int32_t e_max, uint32_t* h_accept_bits,
                         uint8_t* h_errcount, void* d_ws, size_t ws_bytes, int64_t chunk_pairs,
                         void* stream);

/* Accuracy harness: the ground truth of the paper's
 * accuracy study -- exact global edit distance, as Edlib in global mode
 * -- and the false-accept / false-reject tallies of filter
 * decisions (Tables S.2-S.12).  Not on the filtering path.
 *
 * gk_edit_distance: Levenshtein distance of the first len bytes of read p and
 * reference segment p (rows of `stride` bytes, as gk_filter_ascii), bytes
 * compared exactly; Myers' bit-vector algorithm, one thread per pair.
 *  d_dist : n_pairs int32 (written).
 * Errors: GK_ERR_ARG, GK_ERR_LEN, GK_ERR_ALIGN, GK_ERR_CUDA. */
int gk_edit_distance(const uint8_t* d_reads, const uint8_t* d_refs, int64_t stride,
                     int64_t n_pairs, int32_t len, int32_t* d_dist, void* stream);

/* gk_accuracy: for each row r of decisions (threshold d_e_list[r], accept bits
 * at d_accept_bits + r*bits_row_stride, error counts at d_errcount +
 * r*err_row_stride), d_counts[4r .. 4r+3] = {defined pairs, accepted, false
 * accepts (accepted, dist > e), false rejects (rejected, dist <= e)}; pairs
 * with error count 255 (undefined) are left out.
 *  d_e_list : n_rows int32 in device memory.  d_counts : 4*n_rows u64 (written).
 * Errors: GK_ERR_ARG, GK_ERR_ALIGN, GK_ERR_CUDA. */
int gk_accuracy(const uint32_t* d_accept_bits, int64_t bits_row_stride, const uint8_t* d_errcount,
                int64_t err_row_stride, const int32_t* d_dist, int64_t n_pairs,
                const int32_t* d_e_list, int32_t n_rows, uint64_t* d_counts, void* stream);

/* End-to-end from HOST buffers (the paper's "filter time"): the
 * pairs stream through device memory in chunks on two CUDA streams, overlapping
 * the host->device copy of one chunk with the kernels of the next and the
 * device->host copy of the previous one.  Per chunk: gk_encode of both sets,
 * gk_filter at threshold e and, if indices are requested, gk_compact (the
 * accepted pairs handed on to verification).
 *  h_reads, h_refs : n_pairs rows of `stride` bytes in host memory (pinned memory
 *                    gives full PCIe / C2C bandwidth; pageable works).
 *  h_accept_bits   : gk_result_words(n_pairs) u32 in host memory (written) or NULL.
 *  h_errcount      : n_pairs bytes in host memory (written) or NULL.
 *  h_idx, h_n_acc  : ascending indices of the accepted pairs (room for n_pairs
 *                    u32; n_pairs < 2^32) and their number (one u64), or both
 *                    NULL.  At least one of h_accept_bits / h_idx is required.
 *  d_ws            : device scratch of gk_host_workspace_bytes(chunk_pairs, stride,
 *                    len) bytes, 256-byte aligned; chunk_pairs (a multiple of 1024,
 *                    > 0) sets the pipeline granularity.
 *  stream          : the call is ordered after all work already enqueued on it
 *                    (e.g. the producer of d_ws); the pipeline runs on two
 *                    internal streams (created once per host thread and device,
 *                    with a 16-byte pinned count buffer, and reused).
 * Synchronous: returns after the results are in host memory.
 * Errors: as gk_filter_ascii + GK_ERR_WORKSPACE. */
size_t gk_host_workspace_bytes(int64_t chunk_pairs, int64_t stride, int32_t len);
int gk_filter_host(const uint8_t* h_reads, const uint8_t* h_refs, int64_t stride,
                   int64_t n_pairs, int32_t len, int32_t e,
                   uint32_t* h_accept_bits, uint8_t* h_errcount,
                   uint32_t* h_idx, uint64_t* h_n_acc,
                   void* d_ws, size_t ws_bytes, int64_t chunk_pairs, void* stream);

/* Threshold sweep from HOST buffers: every chunk of pairs crosses PCIe and is
 * encoded once, then filtered for every e <= e_max = max(e_list) in one pass
 * (gk_filter_sweep; the paper sweeps e from 0 to 10% of L), and
 * the rows of the requested thresholds are copied back.
 *  e_list          : n_e thresholds (host array), each 0 <= e < len.
 *  h_accept_bits   : n_e * gk_result_words(n_pairs) u32, row t = e_list[t] (written).
 *  h_errcount      : n_e * n_pairs bytes, row t = e_list[t] (written) or NULL.
 *  d_ws            : gk_host_sweep_workspace_bytes(chunk_pairs, stride, len, e_max)
 *                    bytes (e_max = the largest threshold of e_list).
 *  stream          : as gk_filter_host.
 * Synchronous.  Errors: as gk_filter_host. */
size_t gk_host_sweep_workspace_bytes(int64_t chunk_pairs, int64_t stride, int32_t len, int32_t e_max);
int gk_filter_host_sweep(const uint8_t* h_reads, const uint8_t* h_refs, int64_t stride,
                         int64_t n_pairs, int32_t len, const int32_t* e_list, int32_t n_e,
                         uint32_t* h_accept_bits, uint8_t* h_errcount,
                         void* d_ws, size_t ws_bytes, int64_t chunk_pairs, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GATEKEEPER_H */
