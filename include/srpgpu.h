/*
 * srpgpu -- C-ABI of the B200-native SRP-map hot path (sm_100a).
 *
 * The reference (`srpmap`, pure Python/NumPy) has no FFI; its drop-in boundary is
 * the Python API re-exported in srpmap/__init__.py:11-34 and dispatched by
 * cli.evaluate_map (cli.py:170-180).  Each entry point below replaces one of
 * those functions, batched over a leading frame axis.  Conventions:
 *
 *   - every pointer is DEVICE memory owned by the caller (no allocation inside);
 *   - complex arrays are interleaved float32 (re, im), i.e. complex64;
 *   - frame-major layouts: spectra [F][M][K+1], gcc [F][P][K-1], samples [F][S],
 *     maps z [F][J]; `keys` [F] are packed per-frame argmax keys
 *       key = (ordered_f32_bits(z_max) << 32) | (0xFFFFFFFF - i_max)
 *     (largest value, ties to the LOWEST index as np.argmax, srp.py:74-80);
 *     decode with srpgpu_decode_keys;
 *   - work is stream-ordered on `stream` (a cudaStream_t; NULL = legacy default);
 *   - return 0 on success, a negative SRPGPU_ERR_* otherwise; no exception or
 *     C++ type crosses the ABI; srpgpu_last_error() returns the message.
 *     The Python layer maps codes onto the reference's exception classes
 *     (errors.py:4-29): DIMENSION -> DimensionError, VALUE -> ValueError,
 *     CAPACITY -> CapacityError, UNSUPPORTED -> ValueError, LAUNCH -> RuntimeError.
 */
#ifndef SRPGPU_H
#define SRPGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRPGPU_ABI_VERSION 1

typedef void* srpgpu_stream_t; /* cudaStream_t */

#define SRPGPU_OK 0
#define SRPGPU_ERR_DIMENSION (-1)
#define SRPGPU_ERR_VALUE (-2)
#define SRPGPU_ERR_CAPACITY (-3)
#define SRPGPU_ERR_LAUNCH (-4)
#define SRPGPU_ERR_UNSUPPORTED (-5)

/* ---- housekeeping ------------------------------------------------------- */
const char* srpgpu_last_error(void);
int srpgpu_abi_version(void);
/* number of kernels launched through this library since load */
uint64_t srpgpu_launch_count(void);
int srpgpu_device_sync(void);
/* Frontend kernel used by srpgpu_gcc_frames / srpgpu_frames_to_samples*: 0 = by batch
 * size (default), 1 = warp per frame, 2 = a warp per channel / pair task, 3 = the
 * generic block kernel.  All four compute the same values (within fp32 rounding);
 * the choice only changes speed.  Process-wide tuning knob, read at launch. */
int srpgpu_set_frontend_kernel(int32_t which);

/* ---- frontend (srpmap/frontend.py) --------------------------------------- */

/* stft_frame (frontend.py:89-107), frames first_frame .. first_frame+num_frames-1:
 * spectra[f][m][k] = rfft(samples[m][(first+f)*hop : +frame_len] * window)[k], k = 0..K.
 * samples: [M][ld_samples] f32 (num_samples valid per row); window: [frame_len] f32;
 * frame_len a power of two in [4, 16384].  energy (nullable): [F] sum |Y|^2.
 * Out-of-range frames -> SRPGPU_ERR_DIMENSION (the reference's IndexError, :102-105). */
int srpgpu_stft(const float* samples, int32_t num_channels, int64_t num_samples, int64_t ld_samples,
                const float* window, int32_t frame_len, int32_t hop, int64_t first_frame,
                int64_t num_frames, float* spectra, float* energy, srpgpu_stream_t stream);

/* fd_gcc (frontend.py:127-160) on spectra [F][M][K+1]:
 * gcc[f][p][k-1] = Y_m[k] conj(Y_m'[k]) for pairs[p] = (m, m'), k = 1..K-1;
 * weighting 1 (PHAT) divides by max(|raw|, floor), 0 where that is 0;
 * floor_mode 0: floor = floor_value * sum_{m,k=0..K} |Y|^2 of the frame (default
 * floor_value 1e-12, frontend.py:19,154-156); floor_mode 1: floor = floor_value.
 * pairs: device [P][2] int32. */
int srpgpu_fd_gcc(const float* spectra, int64_t num_frames, int32_t num_channels, int32_t half_len,
                  const int32_t* pairs, int32_t num_pairs, int32_t weighting, int32_t floor_mode,
                  double floor_value, float* gcc, srpgpu_stream_t stream);

/* fused stft_frame + fd_gcc: samples -> gcc [F][gcc_ld] complex64 (spectra stay on chip).
 * gcc_ld: complex elements per frame row (0 = P*(K-1); larger pitches are zero-padded).
 * flags bit 0: round the outputs to TF32 (round-to-nearest-even) for srpgpu_srp_map_tc. */
int srpgpu_gcc_frames(const float* samples, int32_t num_channels, int64_t num_samples,
                      int64_t ld_samples, const float* window, int32_t frame_len, int32_t hop,
                      int64_t first_frame, int64_t num_frames, const int32_t* pairs,
                      int32_t num_pairs, int32_t weighting, int32_t floor_mode, double floor_value,
                      float* gcc, int64_t gcc_ld, int32_t flags, srpgpu_stream_t stream);

/* ---- sampling (srpmap/sampling.py) --------------------------------------- */

/* td_gcc_samples(gcc, spec, "ifft") (sampling.py:106-134): per pair the
 * unnormalized real inverse DFT of the two-sided spectrum (bins 0, K zero), lags
 * kept in storage order 0..N_p, -N_p..-1 (sampling.py:62-65) at sample index
 * s = offsets[p] + j.  counts [P], offsets [P+1] are device int32.
 * samples_ld == 0: frame-major samples_out[f][s]; samples_ld >= F: lag-major
 * samples_out[s][f] with row pitch samples_ld (the layout the map kernels read). */
int srpgpu_td_gcc_samples(const float* gcc, int64_t num_frames, int32_t num_pairs, int32_t half_len,
                          const int32_t* counts, const int32_t* offsets, int32_t total_samples,
                          float* samples_out, int64_t samples_ld, srpgpu_stream_t stream);

/* fused stft_frame + fd_gcc + td_gcc_samples: signal -> TD-GCC samples (layout as above). */
int srpgpu_frames_to_samples(const float* samples, int32_t num_channels, int64_t num_samples,
                             int64_t ld_samples, const float* window, int32_t frame_len, int32_t hop,
                             int64_t first_frame, int64_t num_frames, const int32_t* pairs,
                             int32_t num_pairs, int32_t weighting, int32_t floor_mode,
                             double floor_value, const int32_t* counts, const int32_t* offsets,
                             int32_t total_samples, float* samples_out, int64_t samples_ld,
                             srpgpu_stream_t stream);

/* frames_to_samples plus the bf16 hi/lo planes [2][F][cols8] of the samples (the
 * tensor-core interpolation maps' operand), written by the same kernel; cols8 >=
 * total_samples, a multiple of 8.  planes_ld > 0: lag-major planes [2][cols8][planes_ld]
 * instead (planes_ld >= F, a multiple of 8; needs lag-major samples, samples_ld > 0).
 * natural bit 0: sample index in natural lag order -N_p..N_p per pair
 * (srpgpu_interp_map_gather_tc); natural_src [S] int32 maps each natural index to its
 * storage index (used when a non-warp kernel produced the samples).  natural bit 1:
 * fp32 TF32 planes (hi = tf32_rne(x), lo = tf32_rne(x - hi); lag-major only) for
 * srpgpu_interp_map_gather_tf32.  natural bit 2: fp16 planes (hi = f16_rne(x), lo =
 * f16_rne(x - hi); lag-major only, planes_ld a multiple of 64) for
 * srpgpu_interp_map_gather_f16 -- PHAT-weighted samples only (|xi| <= 2(K-1) fits fp16). */
int srpgpu_frames_to_samples_planes(const float* samples, int32_t num_channels, int64_t num_samples,
                                    int64_t ld_samples, const float* window, int32_t frame_len,
                                    int32_t hop, int64_t first_frame, int64_t num_frames,
                                    const int32_t* pairs, int32_t num_pairs, int32_t weighting,
                                    int32_t floor_mode, double floor_value, const int32_t* counts,
                                    const int32_t* offsets, int32_t total_samples, float* samples_out,
                                    int64_t samples_ld, void* planes, int32_t cols8, int64_t planes_ld,
                                    int32_t natural, const int32_t* natural_src, srpgpu_stream_t stream);

/* The whole SSPI chain in one launch (stft_frame + fd_gcc + td_gcc_samples + sspi_map +
 * locate; frontend.py:89-160, sampling.py:106-134, interpolation.py:188-195, srp.py:74-80):
 * signal -> z [F][J] (nullable) and the per-frame argmax index [F] int64 / packed key [F]
 * (each nullable).  The TD-GCC samples never leave shared memory.  The operator is a sliced
 * ELL image of the SparseInterp CSR: candidates in chunks of 32, chunk c's entries at rows
 * sell_chunk_off[c] .. sell_chunk_off[c+1]-1 of sell_cols / sell_vals [rows][32] (sample
 * index uint16, weight f32; padding entries weight 0).  frame_len 256, 512 or 1024;
 * total_samples <= 65535; SRPGPU_ERR_UNSUPPORTED when the frame does not fit in shared memory. */
int srpgpu_frames_to_sspi_map(const float* samples, int32_t num_channels, int64_t num_samples,
                              int64_t ld_samples, const float* window, int32_t frame_len, int32_t hop,
                              int64_t first_frame, int64_t num_frames, const int32_t* pairs, int32_t num_pairs,
                              int32_t weighting, int32_t floor_mode, double floor_value, const int32_t* counts,
                              const int32_t* offsets, int32_t total_samples, const uint16_t* sell_cols,
                              const float* sell_vals, const int32_t* sell_chunk_off, int64_t num_candidates,
                              float* z, int64_t* index, uint64_t* keys, srpgpu_stream_t stream);

/* The SLRI chain in one launch (stft_frame + fd_gcc + td_gcc_samples + slri_map + locate;
 * interpolation.py:178-185): y = fat [R][S] . xi per frame in shared memory, then
 * z = tall . y with the tall factor transposed, tall_t [round16(R)][J] (candidates
 * contiguous; rows R.. zero).
 * Outputs as srpgpu_frames_to_sspi_map; f32 throughout. */
int srpgpu_frames_to_slri_map(const float* samples, int32_t num_channels, int64_t num_samples,
                              int64_t ld_samples, const float* window, int32_t frame_len, int32_t hop,
                              int64_t first_frame, int64_t num_frames, const int32_t* pairs, int32_t num_pairs,
                              int32_t weighting, int32_t floor_mode, double floor_value, const int32_t* counts,
                              const int32_t* offsets, int32_t total_samples, const float* fat, const float* tall_t,
                              int32_t rank, int64_t num_candidates, float* z, int64_t* index, uint64_t* keys,
                              srpgpu_stream_t stream);

/* fused fd_gcc + td_gcc_samples on precomputed spectra [F][M][K+1]. */
int srpgpu_spectra_to_samples(const float* spectra, int64_t num_frames, int32_t num_channels,
                              int32_t half_len, const int32_t* pairs, int32_t num_pairs,
                              int32_t weighting, int32_t floor_mode, double floor_value,
                              const int32_t* counts, const int32_t* offsets, int32_t total_samples,
                              float* samples_out, int64_t samples_ld, srpgpu_stream_t stream);

/* ---- scene synthesis (srpmap/simulate.py) -------------------------------- */

/* synthesize (simulate.py:232-265), room-response part: for every microphone m and image
 * source i (num_images per microphone, image order shared by all microphones)
 *   out[m][n] += gain[m][i] * sum_t taps[m][i][t] * dry[n - start[m][i] - t]   (t < 64)
 * accumulated in image order into direct [M][N] (is_direct[i] != 0) or reverb [M][N];
 * float64 throughout.  start = floor(delay) - 31, taps = the 64-tap fractional-delay
 * kernel, gain = image gain / distance, all computed on the host. */
int srpgpu_render_images(const double* dry, int64_t num_samples, int32_t num_mics, int32_t num_images,
                         const int64_t* start, const double* gain, const double* taps,
                         const int32_t* is_direct, double* direct, double* reverb, srpgpu_stream_t stream);

/* ---- maps (srpmap/interpolation.py, lowrank.py, srp.py) ------------------- */

/* sspi_map (interpolation.py:188-195) and, with a keep-all operator, si_map
 * (:129-136).  samples: lag-major [S][samples_ld] (samples_ld >= F, multiple of 4,
 * 16-byte aligned).  Operator: tiled band image (tiles of 32 candidates, groups of 4):
 * tile t's blob starts at byte tile_offsets[t] of `blob` and holds
 *   meta[P][8] u32 = (record offset << 8) | record count, padded to 16 bytes,
 *   records {u32 sample index, u32 pad[3], f32 weight[4]} for each (pair, group),
 *   pair-major, then group, then ascending sample index;
 * max_pair_records / max_tile_records = largest record count of one (tile, pair) / of one
 * tile (shared-memory staging size).  z [F][J] and keys [F] are each optional (NULL). */
int srpgpu_sspi_map(const float* samples, int64_t samples_ld, int64_t num_frames,
                    int32_t total_samples, int32_t num_pairs, const int64_t* tile_offsets,
                    const void* blob, int64_t num_candidates, int64_t max_pair_records,
                    int64_t max_tile_records, float* z, uint64_t* keys, srpgpu_stream_t stream);

/* Tensor-core engine for the same maps (si_map :129-136 / sspi_map :188-195) when the
 * operator is stored dense (dropped entries = 0).  Operands are bf16 hi/lo plane pairs
 * [2][rows][cols8] (x = hi + lo; cols8 = S rounded up to 8, zero beyond S) made by
 * srpgpu_split_bf16; z ~= Lh.xh + Lh.xl + Ll.xh in fp32 (tcgen05 kind::f16).
 * samples_planes: [2][F][cols8]; op_planes: [2][J][cols8]; z [F][J] and keys [F] are
 * each optional (NULL).  Both plane buffers 16-byte aligned. */
int srpgpu_interp_map_tc(const void* samples_planes, int64_t num_frames, const void* op_planes,
                         int64_t num_candidates, int32_t cols8, float* z, uint64_t* keys,
                         srpgpu_stream_t stream);

/* sspi_map / si_map on the tensor cores for long sample vectors: per-tile gathered lag
 * windows (host layout: paper_2306_08514_b200/tiles.py).  samples_planes: lag-major
 * bf16 planes [2][round8(num_cols)][planes_ld] in natural lag order (planes_ld >= F,
 * multiple of 8); slab_planes [2][num_slabs * 128][64] bf16 (tile operator slabs: 64-lag
 * block b of a tile, half h -> slab 2b + h); group_col [num_blocks * 8] first natural
 * sample index of each 8-lag group; tile_slab / tile_nkb [num_tiles] first 64-lag block
 * and block count of each tile (<= 128); tile_rows [num_tiles][256] candidate index of
 * each tile row (ascending, -1 pad; rows 0-127 half 0);
 * num_ctas persistent CTAs take the work units (group of 8 frame tiles, tile, frame tile)
 * round-robin (num_ctas = the SM count).
 * z [F][J] and keys [F] optional.  With z_tiles the map is written in tile order into
 * z_tiles [F][num_tiles * 256] (full 32-byte sectors) and gathered back to grid order by
 * tile_pos [J] (= tile * 256 + row of each candidate); with z_tiles NULL it is written
 * straight into grid order (no gather pass, but 32-byte sectors shared between tiles are
 * read-modify-written: 2.3x slower at cfg4). */
int srpgpu_interp_map_gather_tc(const void* samples_planes, int64_t num_frames, int32_t num_cols,
                                int64_t planes_ld,
                                const void* slab_planes, int64_t num_slabs, const int32_t* group_col,
                                const int32_t* tile_slab, const int32_t* tile_nkb, const int32_t* tile_rows,
                                int32_t num_tiles, int64_t num_candidates, int32_t num_ctas,
                                const int32_t* tile_pos, float* z_tiles, float* z,
                                uint64_t* keys, srpgpu_stream_t stream);

/* The same map with 3xTF32 operands (FP32-class: hi = tf32_rne(x), lo = tf32_rne(x - hi),
 * z ~= Lh.xh + Lh.xl + Ll.xh accumulated in fp32 by tcgen05 kind::tf32): samples_planes
 * fp32 [2][round8(S)][planes_ld] (planes_ld a multiple of 32, 128-byte aligned; natural lag
 * order), slab_planes fp32 [2][num_slabs * 128][64] (srpgpu_split_tf32 of the slabs);
 * tile_nkb here counts each tile's 16-lag stages (its window rounded up to 16 lags, not to
 * the 64-lag block) and group_col holds 4-lag groups (16 per block); the other arguments
 * as srpgpu_interp_map_gather_tc, except that z_tiles is scratch of round256(F) rows of
 * num_tiles * 256 floats (the CTA-pair kernel stores it in blocks of 32 frames:
 * [frame block][tile][32 frames][256 rows]); with z, z_tiles NULL and tile_pos NULL the tiles
 * are taken to be 256 consecutive candidates each (tile_rows[t][r] = 256 t + r) and the map
 * is stored straight into z with 2D TMA boxes (J % 4 == 0).  Replaces
 * interpolation.py:188-195 (sspi_map) at long sample vectors. */
int srpgpu_interp_map_gather_tf32(const float* samples_planes, int64_t num_frames, int32_t num_cols,
                                  int64_t planes_ld, const float* slab_planes, int64_t num_slabs,
                                  const int32_t* group_col, const int32_t* tile_slab, const int32_t* tile_nkb,
                                  const int32_t* tile_rows, int32_t num_tiles, int64_t num_candidates,
                                  int32_t num_ctas, const int32_t* tile_pos, float* z_tiles, float* z,
                                  uint64_t* keys, srpgpu_stream_t stream);

/* The same map with fp16x3 operands (FP32-class while the operands stay in fp16 range:
 * hi = f16_rne(x), lo = f16_rne(x - hi) carry the same 11 + 11 significant bits as the TF32
 * split; tcgen05 kind::f16 at twice the TF32 rate; TMEM chunks folded into fp32 registers):
 * samples_planes fp16 [2][round8(S)][planes_ld] (planes_ld a multiple of 64, 128-byte
 * aligned, natural lag order; PHAT samples are bounded by 2(K-1)), slab_planes fp16
 * [2][num_slabs * 128][64] = srpgpu_split_f16_rows of the slabs scaled by 1 / z_scale (a
 * power of two; the kernel multiplies the finished sums by z_scale, exactly); group_col
 * holds 8-lag groups (8 per block) and tile_nst counts each tile's 32-lag stages; z_tiles is
 * scratch of round256(F) rows of num_tiles * 256 floats.  CTA pairs (cta_group::2) only.  Replaces interpolation.py:188-195 (sspi_map) / :129-136 (si_map). */
int srpgpu_interp_map_gather_f16(const void* samples_planes, int64_t num_frames, int32_t num_cols,
                                 int64_t planes_ld, const void* slab_planes, int64_t num_slabs,
                                 const int32_t* group_col, const int32_t* tile_slab, const int32_t* tile_nst,
                                 const int32_t* tile_rows, int32_t num_tiles, int64_t num_candidates,
                                 int32_t num_ctas, const int32_t* tile_pos, float z_scale, float* z_tiles,
                                 float* z, uint64_t* keys, srpgpu_stream_t stream);

/* The gather pass of the tile-order scratch alone: z[f][j] = z_tiles[f][tile_pos[j]] after a
 * srpgpu_interp_map_gather_tf32 / _f16 call that was given z_tiles but no z (the two halves of
 * the map stage, so that each can be timed on its own).  blocked != 0: the CTA-pair kernels'
 * scratch layout ([frame block of 32][tile][32 frames][256 rows]); 0: rows of num_tiles * 256. */
int srpgpu_interp_map_untile(const float* z_tiles, int32_t num_tiles, const int32_t* tile_pos,
                             int64_t num_candidates, int64_t num_frames, float* z, int32_t blocked,
                             srpgpu_stream_t stream);

/* srpgpu_split_bf16_rows into fp16 hi / lo planes of scale * x (hi = f16_rne, lo = f16_rne(. - hi)). */
int srpgpu_split_f16_rows(const float* src, int64_t ld_src, int64_t rows, int64_t cols, const int32_t* row_src,
                          float scale, void* dst, int64_t ld_dst, int64_t rows_dst, srpgpu_stream_t stream);

/* srpgpu_split_bf16_rows into fp32 TF32 hi / lo planes (hi = tf32_rne(x), lo = tf32_rne(x - hi)). */
int srpgpu_split_tf32_rows(const float* src, int64_t ld_src, int64_t rows, int64_t cols, const int32_t* row_src,
                           float* dst, int64_t ld_dst, int64_t rows_dst, srpgpu_stream_t stream);

/* row-wise bf16 hi/lo split: dst[p][r][c] for r < rows, c < cols (pitch ld_dst, plane
 * stride rows_dst * ld_dst) from src[row_src[r]][c] (row_src NULL: identity). */
int srpgpu_split_bf16_rows(const float* src, int64_t ld_src, int64_t rows, int64_t cols, const int32_t* row_src,
                           void* dst, int64_t ld_dst, int64_t rows_dst, srpgpu_stream_t stream);

/* srpgpu_split_bf16 with a column source map: dst column c takes source column
 * col_src[c] (NULL: identity). */
int srpgpu_split_bf16_cols(const float* src, int64_t ld_src, int32_t lag_major, int64_t rows, int32_t cols,
                           const int32_t* col_src, void* dst, int32_t cols8, srpgpu_stream_t stream);

/* f32 [rows][cols] (row pitch ld_src; or lag-major src[c * ld_src + r] if lag_major)
 * -> bf16 planes dst[0][r][c] = bf16_rne(x), dst[1][r][c] = bf16_rne(x - hi), pitch
 * cols8 (multiple of 8, zero-filled in [cols, cols8)). */
int srpgpu_split_bf16(const float* src, int64_t ld_src, int32_t lag_major, int64_t rows, int32_t cols,
                      void* dst, int32_t cols8, srpgpu_stream_t stream);

/* frame-major [rows][ld_src] -> lag-major [cols][ld_dst] (zero-filled pad columns). */
int srpgpu_transpose(const float* src, int64_t rows, int64_t cols, int64_t ld_src, float* dst,
                     int64_t ld_dst, srpgpu_stream_t stream);

/* slri_map (interpolation.py:178-185): z = tall (fat xi).  fat [R][S], tall [J][R]
 * f32; samples lag-major [S][samples_ld] (or frame-major [F][S] if samples_ld == 0);
 * work: 17 * F * R floats of scratch (the rank-R intermediate and split-K partials). */
int srpgpu_slri_map(const float* samples, int64_t samples_ld, int64_t num_frames,
                    int32_t total_samples, const float* fat, const float* tall, int32_t rank,
                    int64_t num_candidates, float* work, float* z, uint64_t* keys,
                    srpgpu_stream_t stream);

/* slri_map with the candidate product on the tensor cores: work [F][R] = fat . xi
 * (fp32, work holds 17 * F * R floats as for srpgpu_slri_map), split into bf16 planes
 * work_planes [2][F][cols8], then z = tall . work^T by srpgpu_interp_map_tc against
 * tall_planes [2][J][cols8] (srpgpu_split_bf16 of tall; cols8 >= R, multiple of 8). */
int srpgpu_slri_map_tc(const float* samples, int64_t samples_ld, int64_t num_frames,
                       int32_t total_samples, const float* fat, const void* tall_planes, int32_t rank,
                       int32_t cols8, int64_t num_candidates, float* work, void* work_planes, float* z,
                       uint64_t* keys, srpgpu_stream_t stream);

/* lr_map with the candidate product on the tensor cores; tall2_planes = planes of
 * [2 Re tall, -2 Im tall] ([2][J][cols8], cols8 >= 2R); work 17 * F * 2R floats,
 * work_planes [2][F][cols8]. */
int srpgpu_lr_map_tc(const float* gcc, int64_t num_frames, int32_t gcc_len, const float* fat2,
                     const void* tall2_planes, int32_t rank, int32_t cols8, int64_t num_candidates,
                     float* work, void* work_planes, float* z, uint64_t* keys, srpgpu_stream_t stream);

/* lr_map (lowrank.py:51-57): z = 2 Re(tall (fat psi)).  Complex factors folded
 * into real ones once on the host: fat2 [2R][2PB] with rows r: (Re fat, -Im fat)
 * and R+r: (Im fat, Re fat) interleaved per bin; tall2 [J][2R] = (2 Re tall | -2 Im tall).
 * gcc [F][PB] complex64 (gcc_len = PB); work: 17 * F * 2R floats of scratch. */
int srpgpu_lr_map(const float* gcc, int64_t num_frames, int32_t gcc_len, const float* fat2,
                  const float* tall2, int32_t rank, int64_t num_candidates, float* work, float* z,
                  uint64_t* keys, srpgpu_stream_t stream);

/* srp_map_exact (srp.py:65-71): z = 2 Re(H psi), fp32 SIMT path.  h2 [J][2PB] holds
 * interleaved (Re H, -Im H) per bin so that z = 2 * h2 . (re, im)(psi). */
int srpgpu_srp_map_simt(const float* gcc, int64_t num_frames, int32_t gcc_len, const float* h2,
                        int64_t num_candidates, float* z, uint64_t* keys, srpgpu_stream_t stream);

/* srp_map_exact on the 5th-gen tensor cores (tcgen05.mma kind::tf32, TMEM
 * accumulators, TMA-staged operands): same operands as srpgpu_srp_map_simt, with
 * row pitches gcc_ld / h2_ld (floats) that are multiples of 4 (16 bytes); the K
 * tail and out-of-range rows are zero-filled by TMA.  kind::tf32 truncates fp32
 * operands, so callers pass TF32-rounded (RNE) operands: srpgpu_round_tf32 or
 * srpgpu_gcc_frames(flags=1).  ksplit > 1 splits K into that many slices of whole
 * 16-k-block chunks (for grids with fewer output tiles than SMs: small batches): the
 * partial maps go to work [ksplit][F][J] f32 and a second kernel sums them in slice order
 * and forms the argmax keys; ksplit = 1 needs no work buffer (NULL). */
int srpgpu_srp_map_tc(const float* gcc, int64_t gcc_ld, int64_t num_frames, int32_t gcc_len,
                      const float* h2, int64_t h2_ld, int64_t num_candidates, int32_t ksplit,
                      float* work, float* z, uint64_t* keys, srpgpu_stream_t stream);

/* srp_map_exact with the steering matrix generated on chip (never stored): for
 * candidate i, pair p, bin k: H = exp(j pi k x[i][p] / K), x = xtab [J][P] f32 = dt * fs
 * (srp.py:51-62).  Same tcgen05 GEMM, TMA streams only the TF32-rounded gcc rows
 * (gcc_ld floats per frame, 16-byte pitch).  The operator for grids whose H does not
 * fit in memory (BASELINE cfg4: 164 GB).  split = 1 selects 3xTF32 (near-fp32 accuracy,
 * 3 MMAs per k-step): gcc then holds the hi plane [F][gcc_ld] followed by the lo plane
 * (srpgpu_split_tf32), and the steering residual is generated on chip as well.
 * ksplit / work: split-K as for srpgpu_srp_map_tc. */
int srpgpu_srp_map_tdoa(const float* gcc, int64_t gcc_ld, int64_t num_frames, int32_t num_pairs,
                        int32_t half_len, const float* xtab, int64_t num_candidates, int32_t split,
                        int32_t ksplit, float* work, float* z, uint64_t* keys, srpgpu_stream_t stream);

/* dst = [hi plane rows][lo plane rows]: hi = tf32_rne(src), lo = tf32_rne(src - hi). */
int srpgpu_split_tf32(const float* src, int64_t ld_src, float* dst, int64_t ld_dst, int64_t rows,
                      int64_t cols, srpgpu_stream_t stream);

/* Steering operand from the reference's complex128 matrix (srp.py:51-62; the "conv"
 * payload of an SRPM cache, cache.py:1-19 / cli.py:137-140): src = interleaved
 * (re, im) float64 rows of pitch ld_src complex elements; dst[r][2c] = f32(Re),
 * dst[r][2c+1] = -f32(Im), TF32-rounded (RNE) when tf32 != 0.  Pad columns of dst
 * are not written. */
int srpgpu_c128_to_steering(const void* src, int64_t ld_src, int64_t rows, int64_t cols, float* dst,
                            int64_t ld_dst, int32_t tf32, srpgpu_stream_t stream);

/* dst[r][c] = tf32_rne(src[r][c]) for c < cols, 0 for cols <= c < ld_dst. */
int srpgpu_round_tf32(const float* src, int64_t ld_src, float* dst, int64_t ld_dst, int64_t rows,
                      int64_t cols, srpgpu_stream_t stream);

/* generic fp32 product out[f][i] = alpha sum_k A[i][k] B[f][k] (+ argmax keys). */
int srpgpu_gemm_nt(const float* A, int64_t lda, const float* B, int64_t ldb, float* out, int64_t ldo,
                   int64_t rows_i, int64_t rows_f, int64_t depth, float alpha, uint64_t* keys,
                   srpgpu_stream_t stream);

/* locate (srp.py:74-80) for every frame of z [F][ldz] (first J columns). */
int srpgpu_argmax(const float* z, int64_t num_frames, int64_t num_candidates, int64_t ldz,
                  uint64_t* keys, srpgpu_stream_t stream);

/* unpack keys -> index [F] int64 and/or value [F] f32 (either may be NULL). */
int srpgpu_decode_keys(const uint64_t* keys, int64_t num_frames, int64_t* index, float* value,
                       srpgpu_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SRPGPU_H */
