/*
 * simcov.h -- C ABI of the SIMCoV diffusion stencil on a zero-padded grid
 * (SURVEY.md sec. 8(f) row f4).  Product code; shares nothing with oracle/.
 *
 * What it computes (sec. II-C task 4: "Virus and inflammatory
 * signals diffuse from established sites of infection to neighboring grid
 * points"; sec. VI-D: edge points read "extra points of
 * value 0" padded around the grid instead of going through boundary checks).
 * The paper gives neither the stencil nor its coefficients; DESIGN.md reading
 * R22 fixes them:
 *
 *   A field is an H x W grid of non-negative integer concentrations (uint32).
 *   Its diffusion rate is the fixed-point fraction a / 2^32, 0 <= a <= 2^30.
 *   One step: every cell sends share(v) = floor(v * a / 2^32) (= __umulhi)
 *   to each of its 4 neighbours and keeps the rest:
 *       v'[y][x] = v[y][x] - 4 share(v[y][x]) + share(v[y-1][x]) + share(v[y+1][x])
 *                                              + share(v[y][x-1]) + share(v[y][x+1])
 *   where a neighbour outside the grid is a padding point of value 0 (it
 *   sends nothing; what is sent to it leaves the grid).  Arithmetic is
 *   modulo 2^32; it equals the exact value whenever that stays below 2^32
 *   (e.g. every concentration < 2^31: one step raises a cell by at most
 *   4 * 2^29 over its own value's kept part).
 *   Each field diffuses independently with its own rate; all fields take the
 *   same number of steps.
 *
 * Layout in device memory (the "padded grid", PAPER.md:570 Fig. simcov_boundary(c)):
 *   pitch = simcov_grid_pitch(W) 32-bit words per row (a multiple of 32, so
 *   every row starts on a 128-byte line); H + 2 rows per field; interior cell
 *   (y, x), 0 <= y < H, 0 <= x < W, at word  (y + 1) * pitch + 4 + x.
 *   Every other word of a field is padding and is zero after any simcov_*
 *   call that writes the field.  Fields of one call sit field_stride words
 *   apart (field_stride >= simcov_grid_words(H, W), a multiple of 4).
 *   simcov_pad / simcov_unpad convert from / to dense row-major H x W arrays.
 *
 * Errors: status codes of sw.h (SW_OK, SW_ERR_INVALID_ARGUMENT, SW_ERR_CUDA);
 * nothing is enqueued when a call returns an argument error.  The text of
 * the last error of the calling thread: simcov_last_error_message().
 * All calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 * default stream) on the current device; no call allocates memory.
 */
#ifndef SIMCOV_B200_H
#define SIMCOV_B200_H

#include <stdint.h>

#include "sw.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Most fields one call diffuses (SIMCoV has two: virions, inflammatory signal). */
#define SIMCOV_MAX_FIELDS 8
/* Largest rate: 1/4 in 32-bit fixed point (a cell never sends more than it holds). */
#define SIMCOV_MAX_RATE (1u << 30)

/* Row pitch in 32-bit words of a padded grid W cells wide (W >= 0); -1 if W < 0
 * or too large (W > 2^30). */
int64_t simcov_grid_pitch(int64_t W);

/* Words of one padded field: (H + 2) * simcov_grid_pitch(W); -1 on bad sizes. */
int64_t simcov_grid_words(int64_t H, int64_t W);

/*
 * Dense -> padded: dense holds n_fields row-major H x W uint32 arrays back to
 * back (H*W words each); padded receives them at field_stride words apart,
 * padding zeroed.  Device pointers; the two must not overlap.
 */
sw_status_t simcov_pad(const uint32_t* dense, uint32_t* padded, int64_t H, int64_t W,
                       int32_t n_fields, int64_t field_stride, void* stream);

/* Padded -> dense (the inverse of simcov_pad; padding is not read). */
sw_status_t simcov_unpad(const uint32_t* padded, uint32_t* dense, int64_t H, int64_t W,
                         int32_t n_fields, int64_t field_stride, void* stream);

/*
 * `steps` diffusion steps of n_fields padded fields, in place.
 *   grid     device, n_fields padded fields (field_stride words apart); on
 *            return (stream order) it holds the fields after `steps` steps.
 *            Its padding is (re)zeroed by the call -- whatever the caller
 *            left there is not read as concentration.
 *   scratch  device, same size and layout as grid, not overlapping it; its
 *            contents are overwritten (a ping-pong buffer).
 *   rates    HOST array of n_fields fixed-point rates a (0 <= a <= 2^30).
 *   steps    >= 0; 0 only re-zeroes the padding.
 * Errors: SW_ERR_INVALID_ARGUMENT for null pointers, H or W < 0, n_fields
 * outside [1, SIMCOV_MAX_FIELDS], a rate > 2^30, steps < 0, a field_stride
 * smaller than simcov_grid_words(H, W) or not a multiple of 4, or a
 * misaligned pointer (grid and scratch must be 16-byte aligned);
 * SW_ERR_CUDA if a launch fails.
 */
sw_status_t simcov_diffuse(uint32_t* grid, uint32_t* scratch, int64_t H, int64_t W,
                           int32_t n_fields, int64_t field_stride, const uint32_t* rates,
                           int32_t steps, void* stream);

/* Selects the kernel schedule for later simcov_diffuse calls of this process
 * (measurement and testing; results are identical):
 *   0 = auto (default: up to 8 steps per launch), 1 = one step per launch,
 *   k >= 2 = up to k steps per launch (temporal blocking: a tile held in
 *   registers for k steps), k <= SIMCOV_MAX_TBLOCK.
 * Errors: SW_ERR_INVALID_ARGUMENT for k outside [0, SIMCOV_MAX_TBLOCK]. */
#define SIMCOV_MAX_TBLOCK 8
sw_status_t simcov_set_schedule(int32_t steps_per_launch);

/* Number of kernels the last simcov_diffuse call of this thread enqueued. */
int32_t simcov_last_launch_count(void);

const char* simcov_last_error_message(void);

#ifdef __cplusplus
}
#endif

#endif /* SIMCOV_B200_H */
