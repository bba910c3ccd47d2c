/*
 * fic_b200.h — the C-ABI drop-in boundary of the B200 fractal (PIFS) codec.
 *
 * Every entry point takes plain C types (pointers + sizes), returns an int32
 * error code and never throws.  0 means success; a nonzero code k in 1..18 is
 * (fic::Errc ordinal + 1) of the reference enum (proj/include/fic/error.hpp:10-29),
 * so a C++ or Python wrapper can rebuild `CodecError(Errc(k-1), detail)` with the
 * same "Name: detail" text (proj/src/error.cpp:30-41); the detail string of the
 * last failure on the calling thread is returned by fic_last_error().
 *
 * The reference has no C-ABI today; each function below names the reference
 * interface whose body it replaces.  All compute entry points run on the
 * calling thread's current CUDA device (cudaGetDevice) and block until their
 * results are in the caller's buffers, like the reference calls they replace.
 * There is no CPU fallback: without a usable CUDA device they fail with
 * FIC_ERR_CUDA.
 */
#ifndef FIC_B200_H
#define FIC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes: Errc ordinal + 1 (proj/include/fic/error.hpp:10-29) ---- */
enum {
  FIC_OK = 0,
  FIC_ERR_MALFORMED_HEADER = 1,
  FIC_ERR_UNSUPPORTED_MAXVAL = 2,
  FIC_ERR_TRUNCATED_DATA = 3,
  FIC_ERR_NOT_SQUARE = 4,
  FIC_ERR_NOT_POWER_OF_TWO = 5,
  FIC_ERR_INDIVISIBLE_BY_RANGE = 6,
  FIC_ERR_TOO_SMALL_FOR_DOMAIN = 7,
  FIC_ERR_ODD_SIDE = 8,
  FIC_ERR_SIDE_MISMATCH = 9,
  FIC_ERR_OUT_OF_BOUNDS = 10,
  FIC_ERR_NO_VALID_POSITIONS = 11,
  FIC_ERR_OUT_OF_RANGE = 12,
  FIC_ERR_GEOMETRY = 13,
  FIC_ERR_SCALE_MISMATCH = 14,
  FIC_ERR_DIMENSION_MISMATCH = 15,
  FIC_ERR_NON_CONTRACTIVE = 16,
  FIC_ERR_BAD_PARAMS = 17,
  FIC_ERR_IO = 18,
  /* not part of the reference enum: device-side failures */
  FIC_ERR_CUDA = 100,
  FIC_ERR_INTERNAL = 101
};

/* CodecParams (proj/include/fic/params.hpp:8-24). */
typedef struct fic_params {
  int32_t n;          /* range side, power of two >= 2 */
  int32_t step;       /* domain grid spacing; 0 = track n */
  int32_t s_bits;     /* 1..16 */
  int32_t o_bits;     /* 1..16 */
  double s_max;       /* snapped to milli precision by normalisation */
  double shadow_eps;  /* >= 0 */
} fic_params;

/* RangeMapping (proj/include/fic/encoded_image.hpp:16-26), 32 bytes, fixed layout.
 * (x, y) is the domain origin in pixels; sym is the normative isometry index
 * (proj/include/fic/transforms.hpp:31-40). */
typedef struct fic_mapping {
  int32_t x;
  int32_t y;
  int32_t sym;
  uint32_t qs;
  uint32_t qo;
  int32_t reserved; /* always 0 */
  double residual;  /* collage error contribution, bit-exact with the reference */
} fic_mapping;

/* EncodeStats (proj/include/fic/encoder.hpp:49-53). */
typedef struct fic_stats {
  uint64_t candidates_tested;
  uint64_t shadow_ranges;
  uint64_t shadow_codeblocks;
} fic_stats;

/* LinearFit (proj/include/fic/encoder.hpp:15-19). */
typedef struct fic_linear_fit {
  double s;
  double o;
  double residual;
} fic_linear_fit;

/* QuantizedFit (proj/include/fic/encoder.hpp:24-30). */
typedef struct fic_quantized_fit {
  uint32_t qs;
  uint32_t qo;
  double s;
  double o;
  double residual;
} fic_quantized_fit;

/* Initial raster kinds of DecodeParams (proj/include/fic/decoder.hpp:29). */
enum { FIC_INITIAL_MID_GRAY = 0, FIC_INITIAL_BLACK = 1, FIC_INITIAL_SUPPLIED = 2 };

/* ---- diagnostics ---- */
const char* fic_last_error(void);          /* detail text of the last failure on this thread */
const char* fic_errc_name(int32_t code);   /* errc_name (proj/src/error.cpp:5-27); "Ok" for 0 */
const char* fic_version(void);

/* ---- host-side validation (no device work) ---- */
/* CodecParams::normalized (proj/src/params.cpp:9-23). */
int32_t fic_normalize_params(const fic_params* in, fic_params* out);
/* validate_geometry (proj/src/image.cpp:138-149). */
int32_t fic_validate_geometry(int32_t width, int32_t height, const fic_params* params);

/* ---- encoder (proj/include/fic/encoder.hpp:61-78) ---- */
/* encode_sequential (proj/src/encoder.cpp:344-366): `out` holds (width/n)^2 records,
 * row-major over the range grid (range row outer).  `stats` may be NULL. */
int32_t fic_encode(const uint8_t* image, int32_t width, int32_t height, const fic_params* params,
                   fic_mapping* out, fic_stats* stats);
/* encode_parallel (proj/src/encoder.cpp:368-427): same result for every worker count and
 * chunk geometry; workers/chunk keep their validation (BadParams) and are otherwise unused. */
int32_t fic_encode_parallel(const uint8_t* image, int32_t width, int32_t height,
                            const fic_params* params, int32_t workers, int32_t chunk_w,
                            int32_t chunk_h, fic_mapping* out, fic_stats* stats);
/* encode_range (proj/src/encoder.cpp:332-342): one range at pixel origin (x, y). */
int32_t fic_encode_range(const uint8_t* image, int32_t width, int32_t height, int32_t x, int32_t y,
                         const fic_params* params, fic_mapping* out, fic_stats* stats);
/* Range-sharded encode of one image (north_star multi-GPU path): encodes range rows
 * [row_begin, row_end) of the range grid only; `out` holds (row_end-row_begin)*(width/n)
 * records.  Stats cover the encoded rows only. */
int32_t fic_encode_rows(const uint8_t* image, int32_t width, int32_t height,
                        const fic_params* params, int32_t row_begin, int32_t row_end,
                        fic_mapping* out, fic_stats* stats);
/* Batch of `count` equal-sized images stored back to back (cfg5 volume); `out` holds
 * count * (side/n)^2 records; `stats` (may be NULL) is the sum over images. */
int32_t fic_encode_batch(const uint8_t* images, int32_t count, int32_t width, int32_t height,
                         const fic_params* params, fic_mapping* out, fic_stats* stats);
/* Device-resident encode for benchmarks: `d_image` and `d_out` are device pointers on the
 * current device, work is enqueued on `stream` (cudaStream_t, NULL = default stream) and the
 * call returns without synchronising.  Stats are computed on the host (they depend only on
 * moments) and are final on return.  Use fic_encode for the drop-in path. */
int32_t fic_encode_device(const uint8_t* d_image, int32_t width, int32_t height,
                          const fic_params* params, fic_mapping* d_out, fic_stats* stats,
                          void* stream);

/* Device-resident range-row shard (the multi-GPU split of one image, cfg4): encodes range rows
 * [row_begin, row_end) of the device image into `d_out` ((row_end-row_begin)*(width/n)
 * records, device memory), enqueued on `stream`; every rank holds the whole image and builds
 * the whole (replicated) domain pool.  Synchronises `stream` once (the survivor-list check);
 * stats cover the encoded rows. */
int32_t fic_encode_rows_device(const uint8_t* d_image, int32_t width, int32_t height,
                               const fic_params* params, int32_t row_begin, int32_t row_end,
                               fic_mapping* d_out, fic_stats* stats, void* stream);

/* Device-resident batch (cfg5 volume): `d_images` holds `count` slices back to back,
 * `d_out` count * (side/n)^2 records, both device pointers.  Up to 64 slices are stacked
 * into one encode pass (one pool, one scan over every slice's ranges; each range only
 * meets its own slice's domains), so a volume costs a handful of launches per 64 slices.
 * Synchronises `stream` before returning; stats are the sum over slices. */
int32_t fic_encode_batch_device(const uint8_t* d_images, int32_t count, int32_t width,
                                int32_t height, const fic_params* params, fic_mapping* d_out,
                                fic_stats* stats, void* stream);

/* ---- per-candidate fit pipeline (proj/include/fic/encoder.hpp:32-45), host fp64 ----
 * A block is `side` x `side` samples, row-major (fic::Block, proj/include/fic/transforms.hpp:13-25). */
/* is_shadow (proj/src/encoder.cpp:60-67): *out = 1 iff N*sum(b^2) - sum(b)^2 <= eps. */
int32_t fic_is_shadow(const double* samples, int32_t side, double eps, int32_t* out);
/* least_squares_fit (proj/src/encoder.cpp:69-76): unconstrained fit of b ~ s*a + o.
 * FIC_ERR_SIDE_MISMATCH when side_a != side_b. */
int32_t fic_least_squares_fit(const double* a, int32_t side_a, const double* b, int32_t side_b,
                              double shadow_eps, fic_linear_fit* out);
/* least_squares_clamped (proj/src/encoder.cpp:78-88): s clamped to +-s_max, o re-fitted and
 * clamped to +-255 (params normalised first). */
int32_t fic_least_squares_clamped(const double* a, int32_t side_a, const double* b, int32_t side_b,
                                  const fic_params* params, fic_linear_fit* out);
/* least_squares (proj/src/encoder.cpp:90-102): clamped fit pushed through the quantisers,
 * residual re-scored with the dequantised values. */
int32_t fic_least_squares(const double* a, int32_t side_a, const double* b, int32_t side_b,
                          const fic_params* params, fic_quantized_fit* out);

/* ---- FIC1 container (proj/include/fic/format.hpp:50-70, proj/src/format.cpp:72-185) ----
 * Record packing / unpacking run on the device (one thread per record). */
/* record_layout (format.cpp:78-89): fields[0..6] = x bits, y bits, 3, s_bits, o_bits,
 * positions per axis x, y; *record_bytes = ceil(sum of the widths / 8).  Host only. */
int32_t fic_record_layout(int32_t width, int32_t height, const fic_params* params, int32_t* fields,
                          int32_t* record_bytes);
/* serialize (format.cpp:105-141) of the (width/n)*(height/n) host records: *size gets the byte
 * count; the bytes are written when `out` holds `cap` >= *size bytes (else size query only).
 * FIC_ERR_OUT_OF_RANGE names the first record off the step grid / outside the grid. */
int32_t fic_serialize(const fic_mapping* maps, int32_t width, int32_t height, const fic_params* params,
                      uint8_t* out, int64_t cap, int64_t* size);
/* The same from device records into device memory on `stream` (e.g. rank 0's gathered codes,
 * so only the packed bytes cross to the host); synchronises `stream` for the error check. */
int32_t fic_serialize_device(const fic_mapping* d_maps, int32_t width, int32_t height,
                             const fic_params* params, uint8_t* d_out, int64_t cap, int64_t* size,
                             void* stream);
/* deserialize (format.cpp:143-185): header fields to *width / *height / *params (normalised),
 * the record count to *count; records (residual 0) to `out` when it holds cap >= count. */
int32_t fic_deserialize(const uint8_t* data, int64_t size, int32_t* width, int32_t* height,
                        fic_params* params, fic_mapping* out, int64_t cap, int64_t* count);

/* ---- decoder (proj/include/fic/decoder.hpp:45-63) ---- */
/* decode_step (proj/src/decoder.cpp:39-79) on fp64 rasters of (width*scale)^2 pixels. */
int32_t fic_decode_step(const double* current, int32_t cur_width, int32_t cur_height,
                        const fic_mapping* maps, int32_t width, int32_t height,
                        const fic_params* params, int32_t scale, double* next);
/* decode_traced (proj/src/decoder.cpp:113-128).  `out` holds (width*scale)^2 bytes;
 * `step_rmse` (may be NULL) holds `iterations` doubles; `has_eps`=0 disables the early stop. */
int32_t fic_decode(const fic_mapping* maps, int32_t width, int32_t height, const fic_params* params,
                   int32_t scale, int32_t iterations, int32_t initial_kind, const uint8_t* supplied,
                   int32_t supplied_width, int32_t supplied_height, int32_t has_eps,
                   double convergence_eps, uint8_t* out, double* step_rmse,
                   int32_t* iterations_run);
/* collage_error (proj/src/decoder.cpp:134-140). */
int32_t fic_collage_error(const uint8_t* image, int32_t img_width, int32_t img_height,
                          const fic_mapping* maps, int32_t width, int32_t height,
                          const fic_params* params, double* out);
/* decoded_error_bound (proj/src/decoder.cpp:142-146); host only. */
int32_t fic_decoded_error_bound(double collage_rmse, double s_max, double* out);

/* ---- device selection ---- */
/* Make `device` the current CUDA device of the calling thread for this library's calls
 * (the library links its own CUDA runtime, so a caller's framework-level device choice
 * does not carry over).  Returns FIC_ERR_CUDA for an invalid ordinal. */
int32_t fic_set_device(int32_t device);
int32_t fic_device_count(int32_t* count);

/* ---- instrumentation ---- */
/* Number of this library's kernels launched since load (all devices). */
uint64_t fic_kernel_launch_count(void);
/* Average device time (ms, CUDA events on the launching stream) of the matcher kernel
 * over the calls since the last reset, and the number of timed launches. */
int32_t fic_matcher_timing(double* avg_ms, uint64_t* launches, int32_t reset);
/* Enable/disable per-launch matcher timing (adds four events per encode). */
void fic_set_matcher_timing(int32_t enabled);
/* Average device time (ms) of the full-level tcgen05 scan kernel alone (the dominant kernel:
 * every range x domain x isometry correlation of the encode) and the number of timed launches. */
int32_t fic_scan_timing(double* avg_ms, uint64_t* launches, int32_t reset);
/* The same launches timed from before the scan kernel to after its expand_kernel (the mask
 * records turned into survivor entries).  Reading either accumulator with reset clears both. */
int32_t fic_scan_expand_timing(double* avg_ms, uint64_t* launches, int32_t reset);
/* Device time (ms) of the decode iterations of fic_decode calls without a convergence test
 * (decode_step kernels with the fused step-RMSE partials), their algorithmic bytes
 * (16 B per output pixel and iteration: the next raster written, the current one read) and
 * the number of timed calls; timing is enabled with fic_set_matcher_timing. */
int32_t fic_decode_timing(double* avg_ms, double* avg_bytes, uint64_t* calls, int32_t reset);
/* Device time (ms) of the K1 pool builder (pool_v3_kernel) in timed encodes, its algorithmic
 * bytes per launch (the image read once + the pool written once: per padded domain 2K bytes of
 * fp16 operand, 8*N u16 exact cells and 16 bytes of moments) and the number of timed launches. */
int32_t fic_pool_timing(double* avg_ms, double* avg_bytes, uint64_t* launches, int32_t reset);
/* Survivors (candidates passing the tensor-core bound) per scan level of the calling
 * process's last tcgen05-path encode; returns the number of levels (0 for the CUDA-core path). */
int32_t fic_last_survivors(uint64_t* counts, int32_t max_levels);
/* (test support) K1 read-back for n in {2, 4, 8}: builds the image's domain pool on the device
 * and copies back, per canonical domain d < D, Sq (sum of the 2x2 group sums q), den =
 * N*Sqq - Sq^2 (-1 for flat code blocks: (double)den <= 16*shadow_eps, encoder.cpp:223) and,
 * if `q8` is non-NULL, the exact u16 cells per isometry q8[(d*8 + s)*N + i] = q[perm_s(i)]
 * (encoder.cpp:205-222); `flat_count` gets the flat domains.  With probe_count > 0 it also
 * returns corr[k] = sum_i q8[(domains[k]*8 + syms[k])*N + i] * b_i for range ranges[k] (the
 * survivor evaluation's exact DP2A correlation, encoder.cpp:236-241). */
int32_t fic_debug_pool(const uint8_t* image, int32_t width, int32_t height, const fic_params* params,
                       int64_t* sq, int64_t* den, uint16_t* q8, uint64_t* flat_count,
                       int32_t probe_count, const int32_t* ranges, const int32_t* domains,
                       const int32_t* syms, int64_t* corr);
/* (diagnostics) clock64 stamps of scan CTA 0's first 256 tiles recorded under FIC_DEBUG=32:
 * per tile 51 slots (MMA issuer before/after the TMEM-buffer wait and after the pool tile landed,
 * each of the 16 epilogue warps releasing the tile, finishing it, and past its per-range test).
 * Copies up to n values. */
int32_t fic_debug_trace(int64_t* out, int32_t n);

#ifdef __cplusplus
}
#endif

#endif /* FIC_B200_H */
