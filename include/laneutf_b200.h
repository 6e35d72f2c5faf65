/*
 * laneutf_b200.h -- C ABI of liblaneutf_b200.so, the B200 (sm_100a) engine
 * behind the reference's reserved ``native`` engine slot.
 *
 * Reference interface each entry point replaces (paths under
 * /root/reference/pkg/src/laneutf/):
 *
 *   lu_utf8_to_utf16le   engine.transcode(UTF8_TO_UTF16, ...)   engine.py:178-209
 *                        (native branch that raises at engine.py:194-200);
 *                        semantics of scalar.transcode_utf8_to_utf16le,
 *                        scalar.py:46-105
 *   lu_utf16le_to_utf8   engine.transcode(UTF16_TO_UTF8, ...)   engine.py:178-209;
 *                        semantics of scalar.transcode_utf16le_to_utf8,
 *                        scalar.py:108-147
 *   lu_validate_utf8     engine.validate(UTF8_TO_UTF16, ...)    engine.py:226-240;
 *                        scalar.validate_utf8, scalar.py:150-197
 *   lu_validate_utf16le  engine.validate(UTF16_TO_UTF8, ...)    engine.py:226-240;
 *                        scalar.validate_utf16le, scalar.py:200-217
 *   lu_utf16_length_from_utf8    scalar.utf16_length_from_utf8,
 *                        scalar.py:220-225 (status + exact word count)
 *   lu_utf8_length_from_utf16le  scalar.utf8_length_from_utf16le,
 *                        scalar.py:228-233 (status + exact byte count)
 *   lu_utf8_char_count   scalar.utf8_char_count, scalar.py:246-248
 *   lu_utf16le_char_count scalar.utf16le_char_count, scalar.py:251-257
 *   lu_utf8_to_utf16be / lu_utf16be_to_utf8 / lu_validate_utf16be
 *                        the CLI's utf16be formats, cli.py:90-94, 113-114
 *   lu_batch_*           many independent cases per launch: the difftest
 *                        campaign / triple sweep, difftest.py:90-104
 *   lu_workspace_bytes   (new) sizing helper; the output sizing rule is
 *                        engine.worst_case_output_bytes, engine.py:171-175
 *   lu_device_supported  engine.detect() capability probe, engine.py:141-153
 *
 * Conventions
 *   - All data pointers are DEVICE pointers; every call is stream-ordered on
 *     ``stream`` and returns as soon as the work is enqueued.
 *   - ``res`` is a device-resident lu_outcome written by the kernel:
 *     {status, consumed, written} with the reference's TranscodeOutcome
 *     meaning (outcome.py:57-83): status 0 OK, 1 MALFORMED_INPUT;
 *     ``consumed`` counts input units (bytes / 16-bit words) before the first
 *     invalid unit (== the error offset); ``written`` counts output units
 *     (16-bit words / bytes).  Validators always report written = 0; the
 *     length functions report the output length of the whole input in
 *     ``written`` when it is valid (0 when malformed: the reference raises).
 *   - Output buffers must hold the worst case (1 word per UTF-8 byte, 3 bytes
 *     per UTF-16 word).  Exactly out[0 .. written) is written; nothing past
 *     it (the reference's canary contract).
 *   - ``ws`` is caller-owned device scratch of at least
 *     lu_workspace_bytes(op, n_units) bytes, 8-byte aligned, any contents
 *     (each call zeroes what it uses on its stream); the library allocates
 *     nothing.  Its only global state is a mutex-protected per-device cache
 *     (kernel attributes, resident capacity).  One workspace must not be
 *     shared by calls that may run concurrently; calls on disjoint buffers
 *     may run concurrently on any streams and threads.
 *   - Concurrency with other kernels: the transcode kernels are persistent
 *     (grid <= resident capacity) but do NOT require their CTAs to be
 *     co-resident -- the tile-ordering scanner is the first CTA to start and
 *     every wait is on work claimed by running CTAs -- so they make progress
 *     when other work holds SMs.  A spin-wait that sees no progress for 10 s
 *     of GPU time traps (a launch error) rather than hanging.
 *   - Return value 0 = enqueued; negative = error, message in lu_last_error()
 *     (thread-local).  Malformed input is NOT an error: it is a status.
 */
#ifndef LANEUTF_B200_H
#define LANEUTF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *lu_stream_t; /* == cudaStream_t */

typedef struct {
    int32_t status; /* 0 ok, 1 malformed-input, 2 output-too-small (unused) */
    int32_t pad;
    uint64_t consumed;
    uint64_t written;
} lu_outcome;

enum {
    LU_OP_UTF8_TO_UTF16LE = 0,
    LU_OP_UTF16LE_TO_UTF8 = 1,
    LU_OP_VALIDATE_UTF8 = 2,
    LU_OP_VALIDATE_UTF16LE = 3,
    LU_OP_UTF16_LENGTH_FROM_UTF8 = 4,
    LU_OP_UTF8_LENGTH_FROM_UTF16LE = 5,
    LU_OP_UTF8_CHAR_COUNT = 6,
    LU_OP_UTF16LE_CHAR_COUNT = 7,
    LU_OP_UTF8_TO_UTF16BE = 8,
    LU_OP_UTF16BE_TO_UTF8 = 9,
    LU_OP_VALIDATE_UTF16BE = 10
};

enum {
    LU_OK = 0,
    LU_ERR_INVALID = -1,   /* null / misaligned pointer, bad size */
    LU_ERR_WORKSPACE = -2, /* ws_bytes < lu_workspace_bytes(...) */
    LU_ERR_CAPACITY = -3,  /* output capacity below the worst case */
    LU_ERR_CUDA = -4       /* CUDA runtime error (see lu_last_error) */
};

int lu_utf8_to_utf16le(const uint8_t *in, uint64_t n_bytes, uint16_t *out, uint64_t out_cap_words, void *ws,
                       uint64_t ws_bytes, lu_outcome *res, lu_stream_t stream);

int lu_utf16le_to_utf8(const uint16_t *in, uint64_t n_words, uint8_t *out, uint64_t out_cap_bytes, void *ws,
                       uint64_t ws_bytes, lu_outcome *res, lu_stream_t stream);

int lu_validate_utf8(const uint8_t *in, uint64_t n_bytes, void *ws, uint64_t ws_bytes, lu_outcome *res,
                     lu_stream_t stream);

int lu_validate_utf16le(const uint16_t *in, uint64_t n_words, void *ws, uint64_t ws_bytes, lu_outcome *res,
                        lu_stream_t stream);

/* UTF-16BE variants: identical outcomes to the LE calls on the byte-swapped
 * buffer (the reference swaps the whole buffer in its CLI, cli.py:90-94,
 * 113-114, with engine.swap_utf16_byte_order, engine.py:243-250); here the
 * swap is fused into K1's compaction and K2/K4's load. */
int lu_utf8_to_utf16be(const uint8_t *in, uint64_t n_bytes, uint16_t *out, uint64_t out_cap_words, void *ws,
                       uint64_t ws_bytes, lu_outcome *res, lu_stream_t stream);

int lu_utf16be_to_utf8(const uint16_t *in, uint64_t n_words, uint8_t *out, uint64_t out_cap_bytes, void *ws,
                       uint64_t ws_bytes, lu_outcome *res, lu_stream_t stream);

int lu_validate_utf16be(const uint16_t *in, uint64_t n_words, void *ws, uint64_t ws_bytes, lu_outcome *res,
                        lu_stream_t stream);

/* Validate and count in one pass (the validators plus a per-warp reduction). */
int lu_utf16_length_from_utf8(const uint8_t *in, uint64_t n_bytes, void *ws, uint64_t ws_bytes, lu_outcome *res,
                              lu_stream_t stream);

int lu_utf8_length_from_utf16le(const uint16_t *in, uint64_t n_words, void *ws, uint64_t ws_bytes, lu_outcome *res,
                                lu_stream_t stream);

/* Character counts (no validation); *count is a device uint64. */
int lu_utf8_char_count(const uint8_t *in, uint64_t n_bytes, void *ws, uint64_t ws_bytes, uint64_t *count,
                       lu_stream_t stream);

int lu_utf16le_char_count(const uint16_t *in, uint64_t n_words, void *ws, uint64_t ws_bytes, uint64_t *count,
                          lu_stream_t stream);

/* Batched independent cases (the differential campaign / byte-triple sweep
 * through the GPU; reference harness difftest.py:90-104):
 * case i = units [offsets[i], offsets[i+1]) of ``data`` (bytes or 16-bit
 * words), offsets non-decreasing, n_cases + 1 device uint64 entries.
 * res[i] = case i's lu_outcome; case i's output is written at its worst-case
 * slot: out + offsets[i] (words) for UTF-8 -> UTF-16LE, out + 3 * offsets[i]
 * (bytes) for UTF-16LE -> UTF-8, exactly res[i].written units.  No workspace. */
int lu_batch_utf8_to_utf16le(const uint8_t *data, const uint64_t *offsets, uint32_t n_cases, uint16_t *out,
                             lu_outcome *res, lu_stream_t stream);

int lu_batch_utf16le_to_utf8(const uint16_t *data, const uint64_t *offsets, uint32_t n_cases, uint8_t *out,
                             lu_outcome *res, lu_stream_t stream);

int lu_batch_validate_utf8(const uint8_t *data, const uint64_t *offsets, uint32_t n_cases, lu_outcome *res,
                           lu_stream_t stream);

int lu_batch_validate_utf16le(const uint16_t *data, const uint64_t *offsets, uint32_t n_cases, lu_outcome *res,
                              lu_stream_t stream);

uint64_t lu_workspace_bytes(int op, uint64_t n_units);

int lu_device_supported(int device);

/* Input bytes per transcode tile (the unit the central scanner orders; the
 * transcode workspace holds one 8-byte status word per tile).  Informational:
 * callers never need to align anything to it. */
int lu_tile_bytes(void);

const char *lu_last_error(void);

const char *lu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LANEUTF_B200_H */
