/*
 * sw.h -- C ABI of the B200-native batched Smith-Waterman (affine / Gotoh)
 * library.  Product code; shares nothing with oracle/.
 *
 * What a batch computes (sec. II-B1, and the affine
 * gap state of PAPER.md:507 / 713-714; tie rules are DESIGN.md readings
 * R5/R6 = SURVEY.md sec. 8(c) C-4/C-5):
 *
 *   For every pair p, query q = queries[q_offsets[p] .. q_offsets[p+1])
 *   (matrix rows i) and reference r = refs[r_offsets[p] .. r_offsets[p+1])
 *   (matrix columns j):
 *     E[i][j] = max(E[i][j-1] + gap_extend, H[i][j-1] + gap_open)
 *     F[i][j] = max(F[i-1][j] + gap_extend, H[i-1][j] + gap_open)
 *     H[i][j] = max(0, H[i-1][j-1] + s(q_i, r_j), E[i][j], F[i][j])
 *   with H = 0 and E = F = -inf on the borders.  A gap of length k scores
 *   gap_open + (k-1)*gap_extend.
 *     score = S = max H                      (forward pass)
 *     (q_end, r_end) = lexicographically smallest (r_end, q_end) with H = S
 *     (q_start, r_start) from the same recurrence on the reversed prefixes
 *       reverse(q[0..q_end]) x reverse(r[0..r_end]): the lexicographically
 *       smallest reversed (j', i') with H' = S (reverse pass, PAPER.md:153/165,
 *       "two CUDA kernels" PAPER.md:230).
 *   Coordinates are 0-based, inclusive, relative to each sequence.
 *   S == 0 (including an empty sequence)      -> (0, -1, -1, -1, -1)
 *   invalid pair (symbol outside the alphabet,
 *   negative length, length > SW_MAX_SEQ_LEN)  -> (-1, -1, -1, -1, -1)
 *
 * Alphabets (reading R10): DNA = A C G T; protein = the 24 BLOSUM62
 * symbols A R N D C Q E G H I L K M F P S T W Y V B Z X *; both
 * case-insensitive.  Protein always uses the built-in NCBI BLOSUM62.
 *
 * Threading: one host thread and one stream per handle at a time; a handle
 * is bound to the device given to sw_init.  No function prints, throws or
 * exits; errors are status codes (text via sw_last_error_message).
 */
#ifndef SW_B200_H
#define SW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SW_ABI_VERSION 1

/* Longest sequence (either role) the library aligns; longer pairs are
 * per-pair errors.  Positions fit 16 bits in the packed argmax key. */
#define SW_MAX_SEQ_LEN 65535

typedef struct sw_context* sw_handle_t;

typedef enum {
    SW_OK = 0,
    SW_ERR_INVALID_ARGUMENT = 1, /* null handle/pointer, n_pairs < 0, ...            */
    SW_ERR_INVALID_SCORING = 2,  /* preconditions on sw_scoring_t violated          */
    SW_ERR_CUDA = 3,             /* a CUDA runtime call failed (see last error msg) */
    SW_ERR_OUT_OF_MEMORY = 4,    /* workspace allocation failed                     */
    SW_ERR_WRONG_DEVICE = 5,     /* current device differs from the handle's        */
    SW_ERR_BAD_PAIRS = 6,        /* sw_batch_status: >= 1 pair was invalid          */
    SW_ERR_INTERNAL = 7          /* a device self-check failed (never expected)     */
} sw_status_t;

typedef enum { SW_ALPHABET_DNA = 0, SW_ALPHABET_PROTEIN = 1 } sw_alphabet_t;

/* Scoring (host struct, copied at the call).  Preconditions, checked
 * synchronously (SW_ERR_INVALID_SCORING, nothing enqueued):
 *   -32768 <= gap_open < 0  and  gap_open <= gap_extend <= 0
 *   DNA: 0 < match <= 32767  and  -32768 <= mismatch < match
 * (reading R3; "arbitrarily determined" scores). */
typedef struct {
    int32_t alphabet;   /* sw_alphabet_t                                       */
    int32_t match;      /* DNA only: s(a, a)                                   */
    int32_t mismatch;   /* DNA only: s(a, b), a != b                           */
    int32_t gap_open;   /* score of the first residue of a gap (negative)      */
    int32_t gap_extend; /* score of each further residue of the same gap       */
} sw_scoring_t;

/* Output arrays: caller-owned DEVICE memory, n_pairs int32 each, fully
 * overwritten by sw_align_batch. */
typedef struct {
    int32_t* score;
    int32_t* q_end;
    int32_t* r_end;
    int32_t* q_start;
    int32_t* r_start;
} sw_result_t;

/*
 * Pass selection (the paper's V0-style one-kernel
 * mode): SW_MODE_FULL (default) runs the forward and the
 * reverse pass; SW_MODE_END_ONLY runs the forward pass only -- score, q_end
 * and r_end are exact as in FULL mode, q_start / r_start are not written (the
 * sw_result_t pointers may then be NULL).  Flag SW_MODE_AFFINE_ONLY (may be
 * OR-ed with either) keeps linear-gap scorings (gap_open == gap_extend) on the
 * affine kernels instead of the two-state linear-gap kernels (PAPER.md:161-163:
 * the gap scores are free parameters; results are identical either way -- the
 * flag exists for comparison and testing).  Flag SW_MODE_TB_INT32 keeps every
 * sw_traceback pair on the int32 path kernel instead of the s16x2 one (two DNA
 * pairs per warp; identical paths -- comparison and testing).  Flag
 * SW_MODE_POISON (debugging and tests) makes every later call first fill the
 * caller's output arrays and the handle's internal workspace (stripe hand-off
 * rows, work lists, reverse-pass metadata, path scratch) with poison bytes
 * (0x7f / 0xff), so any value a call reads or returns without having written
 * it in that call shows up as a wrong result instead of a stale plausible
 * one; results are unchanged, calls are slower.  Applies to every later call
 * on the handle.  Flag SW_MODE_NO_BAND keeps every reverse-pass pair on the
 * row-sweep kernels instead of the banded reverse kernels (DNA pairs whose
 * score-S paths fit 32 / 64 diagonals; identical results --
 * comparison and testing); batches (host-call chunks) of fewer than 16,384
 * pairs use the row-sweep kernels anyway (too few work items to fill the GPU)
 * unless flag SW_MODE_BAND_ALWAYS is set (testing).  Errors:
 * SW_ERR_INVALID_ARGUMENT for an unknown mode bit.
 */
typedef enum { SW_MODE_FULL = 0, SW_MODE_END_ONLY = 1, SW_MODE_AFFINE_ONLY = 2, SW_MODE_TB_INT32 = 4,
               SW_MODE_POISON = 8, SW_MODE_NO_BAND = 16, SW_MODE_BAND_ALWAYS = 32 } sw_mode_t;
sw_status_t sw_set_mode(sw_handle_t h, int32_t mode);

/*
 * Alignment paths (reading R20).  For a
 * batch already aligned with sw_align_batch / sw_align_batch_host (the same
 * inputs; `res` = its five result arrays in DEVICE memory, full mode), write
 * each pair's alignment as ops from start to end: 'M' an aligned pair, 'I' a
 * query residue against a gap, 'D' a reference residue against a gap.  The
 * path is the optimal global affine alignment of q[q_start..q_end] and
 * r[r_start..r_end] (its score is the pair's S); among several, the one whose
 * op string read from the end is lexicographically greatest with M > I > D
 * (SPEC.md's diagonal > up > left traceback).
 *   queries .. r_offsets, n_pairs, scoring   as for sw_align_batch (DEVICE)
 *   ops     DEVICE uint8, (q_offsets[n]-q_offsets[0]) + (r_offsets[n]-r_offsets[0])
 *           bytes; pair p's ops start at (q_offsets[p]-q_offsets[0]) +
 *           (r_offsets[p]-r_offsets[0]) (a path has at most n_p + m_p ops)
 *   n_ops   DEVICE int32[n_pairs]: op count; 0 when S == 0; -1 for an invalid
 *           pair (score -1)
 * Enqueued on `stream`; synchronises on it once (the batch's largest interval
 * sizes the scratch: one direction word per 5 cells of it per resident warp).
 */
sw_status_t sw_traceback(sw_handle_t h,
                         const uint8_t* queries, const int64_t* q_offsets,
                         const uint8_t* refs, const int64_t* r_offsets,
                         int64_t n_pairs, const sw_scoring_t* scoring,
                         const sw_result_t* res, uint8_t* ops, int32_t* n_ops, void* stream);

/* Create a handle bound to CUDA device `device`.  Allocates no large memory;
 * the workspace grows on demand and is reused across calls. */
sw_status_t sw_init(sw_handle_t* handle, int device);

/*
 * Align a batch (forward + reverse pass).
 *   queries, refs     DEVICE uint8 ASCII bytes (CSR payloads)
 *   q_offsets,
 *   r_offsets         DEVICE int64, n_pairs + 1 entries each, non-decreasing;
 *                     pair p uses [off[p], off[p+1]).  Offsets are relative to
 *                     the payload pointers; off[0] need not be 0.
 *   n_pairs           >= 0 (0 is a no-op)
 *   scoring           HOST pointer, copied
 *   out               HOST struct of DEVICE pointers (see sw_result_t)
 *   stream            a cudaStream_t (NULL = legacy default stream)
 * Work is enqueued on `stream`; inputs and outputs must stay untouched until
 * it completes.  Asynchrony:
 *   - after sw_reserve, a batch within the reservation is enqueued without any
 *     host round trip: the call returns at once and can be captured into a
 *     CUDA graph.  A batch beyond the reservation (payload, pair count, or a
 *     sequence longer than the reserved lengths) and malformed offsets are
 *     detected on the device: every output is -1 and sw_batch_status returns
 *     SW_ERR_INVALID_ARGUMENT / SW_ERR_BAD_PAIRS (count -1).
 *   - without a reservation, the call synchronises on `stream` once (to read
 *     the per-batch length statistics that size the launches; the first call
 *     of a handle, or one whose payload outgrows the handle's code buffers,
 *     also reads the payload extents first), so it returns after earlier work
 *     on `stream` is done but before this batch's kernels finish; malformed
 *     offsets return SW_ERR_INVALID_ARGUMENT (every output -1).
 * Per-pair errors do not fail the call: they appear as -1 sentinels and are
 * counted by sw_batch_status.
 */
sw_status_t sw_align_batch(sw_handle_t h,
                           const uint8_t* queries, const int64_t* q_offsets,
                           const uint8_t* refs, const int64_t* r_offsets,
                           int64_t n_pairs, const sw_scoring_t* scoring,
                           const sw_result_t* out, void* stream);

/*
 * Reserve the handle's workspace for batches of up to max_pairs pairs,
 * max_query_bytes / max_ref_bytes payload bytes (q_offsets[n]-q_offsets[0],
 * r_offsets[n]-r_offsets[0]) and sequences of up to max_query_len /
 * max_ref_len residues (<= SW_MAX_SEQ_LEN).  Afterwards sw_align_batch (and
 * sw_align_query_db once its broadcast buffer exists) never synchronises for a
 * batch with n_pairs <= max_pairs: launches are sized from the reservation
 * and the device-side counts.  Synchronises the device; may be called again
 * (the workspace only grows).  Errors: SW_ERR_INVALID_ARGUMENT (bounds out of
 * range), SW_ERR_OUT_OF_MEMORY, SW_ERR_WRONG_DEVICE.
 */
sw_status_t sw_reserve(sw_handle_t h, int64_t max_pairs, int64_t max_query_bytes, int64_t max_ref_bytes,
                       int32_t max_query_len, int32_t max_ref_len);

/*
 * One query against a database of references (the
 * paper's problem statement, with A fixed): results are
 * those of sw_align_batch on the pairs (query, refs[r_offsets[p] ..
 * r_offsets[p+1])), p = 0 .. n_refs - 1, q coordinates relative to the query.
 *   query             DEVICE uint8 ASCII, n bytes (n >= 0)
 *   refs, r_offsets,
 *   n_refs, scoring,
 *   out, stream       as for sw_align_batch (n_refs pairs)
 * The query is broadcast on `stream` into a handle-owned device buffer of
 * n * n_refs bytes (the batch path then packs and profiles it like any other
 * query).  Errors as for sw_align_batch; SW_ERR_INVALID_ARGUMENT for n < 0 or
 * a NULL query with n > 0.
 */
sw_status_t sw_align_query_db(sw_handle_t h,
                              const uint8_t* query, int64_t n,
                              const uint8_t* refs, const int64_t* r_offsets,
                              int64_t n_refs, const sw_scoring_t* scoring,
                              const sw_result_t* out, void* stream);

/*
 * Same computation with HOST buffers (pinned memory recommended): copies the
 * inputs to handle-owned device staging buffers, aligns, and copies the five
 * result arrays to the HOST pointers in `out_host`.  Synchronous: returns
 * after the results are on the host.  This is the end-to-end entry point.
 */
sw_status_t sw_align_batch_host(sw_handle_t h,
                                const uint8_t* queries, const int64_t* q_offsets,
                                const uint8_t* refs, const int64_t* r_offsets,
                                int64_t n_pairs, const sw_scoring_t* scoring,
                                const sw_result_t* out_host, void* stream);

/*
 * Asynchronous HOST-buffer entry point for a stream of batches (the serving
 * loop): enqueues this batch's host->device copies on a handle-owned copy
 * stream, the alignment on `stream`, and the device->host result copies on a
 * second handle-owned copy stream, and returns without waiting.  Two batches
 * can be in flight: while batch i is aligned on `stream`, batch i+1's inputs
 * are copied in (double-buffered staging), so a stream of batches runs at the
 * alignment's rate rather than alignment + transfer.  Batches are aligned in
 * submission order.  The caller keeps every host buffer of a submitted batch
 * (inputs and out_host) untouched until sw_wait returns.  Arguments as for
 * sw_align_batch_host (q_offsets / r_offsets are read on the host during the
 * call: validation and work estimates); the same validation errors are
 * returned synchronously, before anything is enqueued.
 */
sw_status_t sw_submit_host(sw_handle_t h,
                           const uint8_t* queries, const int64_t* q_offsets,
                           const uint8_t* refs, const int64_t* r_offsets,
                           int64_t n_pairs, const sw_scoring_t* scoring,
                           const sw_result_t* out_host, void* stream);

/* Wait until every batch submitted with sw_submit_host is on the host and make
 * `stream` (the one passed to sw_submit_host) wait for it too. */
sw_status_t sw_wait(sw_handle_t h);

/* Synchronise the handle's last batch and report how many pairs were
 * invalid.  Returns SW_OK, SW_ERR_BAD_PAIRS (count > 0; -1 for malformed
 * offsets), SW_ERR_INVALID_ARGUMENT (a reserved call's batch beyond the
 * reservation) or SW_ERR_INTERNAL (a device self-check, incl. sw_traceback's
 * path walks since the previous sw_batch_status). */
sw_status_t sw_batch_status(sw_handle_t h, int64_t* n_bad_pairs);

/* Synchronise outstanding work, release the workspace and the handle. */
sw_status_t sw_free(sw_handle_t h);

const char* sw_status_string(sw_status_t s);
const char* sw_last_error_message(sw_handle_t h);

/*
 * Cell-count shard plan (host only, no device): cut pairs [0, n_pairs) into
 * n_shards contiguous ranges of near-equal cost sum n_p*m_p (pairs with
 * n_p*m_p == 0 cost 1).  q_offsets_host / r_offsets_host are HOST arrays of
 * n_pairs + 1 entries; shard_begin receives n_shards + 1 indices with
 * shard_begin[0] = 0 and shard_begin[n_shards] = n_pairs.
 */
sw_status_t sw_plan_shards(const int64_t* q_offsets_host, const int64_t* r_offsets_host,
                           int64_t n_pairs, int32_t n_shards, int64_t* shard_begin);

/* ---- instrumentation ------------------------------------------------ */

/* Stage timers (CUDA events on the batch's stream).  Enable before a batch;
 * read after it completes (sw_get_stage_ms synchronises on the last batch). */
#define SW_STAGE_PACK 0      /* validation + ASCII -> codes + length stats       */
#define SW_STAGE_SORT 1      /* forward length binning (radix sort)              */
#define SW_STAGE_FWD 2       /* forward wavefront kernel(s)  <- dominant kernel  */
#define SW_STAGE_MID 3       /* finish_fwd + reverse binning                     */
#define SW_STAGE_REV 4       /* reverse wavefront kernel(s)                      */
#define SW_STAGE_FINISH 5    /* finish_rev                                       */
#define SW_STAGE_COUNT 6
sw_status_t sw_enable_stage_timing(sw_handle_t h, int enable);
sw_status_t sw_get_stage_ms(sw_handle_t h, float ms[SW_STAGE_COUNT]);

/* Number of kernel launches the last batch enqueued (own kernels + CUB
 * sort kernels counted separately). */
sw_status_t sw_last_launch_count(sw_handle_t h, int32_t* own_kernels, int32_t* library_kernels);

/* Forward/reverse cell counts of the last batch (after sw_batch_status or a
 * stream sync): forward = sum n*m over valid pairs; padded = cells the
 * wavefront actually swept (rows padded to the stripe, columns to the work
 * item's longest reference, plus fill/drain). */
sw_status_t sw_last_cell_counts(sw_handle_t h, int64_t* forward_cells, int64_t* swept_cells);

/* Cells the reverse wavefront of the last batch swept (work items' rows x
 * columns up to the early stop, incl. fill/drain).  Same synchronisation as
 * sw_last_cell_counts. */
sw_status_t sw_last_reverse_cells(sw_handle_t h, int64_t* swept_cells);

/*
 * DPX cell-update roofline probe: runs the minimal
 * s16x2 Gotoh cell-pair mix (3 VIADDMNMX.S16x2 + 1 VIMNMX.S16x2 + 1
 * VIADD.16x2 + 1/2 VIMNMX3.S16x2) on independent register chains on every
 * SM for ~`milliseconds`, on `stream`.  Returns cell updates per second
 * (2 per cell-pair step) in *cups.  Synchronous.
 */
sw_status_t sw_dpx_peak(int device, double milliseconds, double* cups, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SW_B200_H */
