/*
 * ddcca.h — C ABI of the B200-native DDCCANet fit/transform path.
 *
 * The reference (ddccanet 0.1.0, pure Python/numpy) has no native FFI; its
 * boundary is the Python API of cascade/moments/solver/encoder/pipeline.
 * Every entry point below replaces one reference function (file:line under
 * /root/reference/pkg/src/ddccanet/) and is bound from Python with ctypes
 * (paper_2209_13027_b200/_native.py; see INTEGRATION.md for the stub a
 * reference maintainer would add).
 *
 * Conventions
 *   - All array arguments are DEVICE pointers (sm_100a, same CUDA context as
 *     the caller), except where a name ends in `_host`.
 *   - `stream` is a cudaStream_t passed as void*; all work is stream-ordered
 *     and asynchronous unless stated. The library keeps no global mutable
 *     state: scratch memory is passed in (`ws`, `ws_bytes`), so calls are
 *     re-entrant across streams and threads.
 *   - Return codes: DDCCA_OK, DDCCA_ESHAPE (reference ShapeError),
 *     DDCCA_ECONFIG (ConfigError), DDCCA_ENUMERICAL (NumericalError),
 *     DDCCA_ECUDA (launch/runtime failure). ddcca_last_error() returns a
 *     thread-local message for the last failing call on this thread.
 *   - Moment payload (one "accumulator", float64, length ddcca_payload_len):
 *       [ c11 (d*d) | c22 (d*d) | s1 (d*C, row-major d x C) | s2 (d*C) |
 *         g1 (d) | g2 (d) | patch_count (1) | per_class_count (C) ]
 *     i.e. the fields of MomentAccumulator (moments.py:26-48). Counts are
 *     stored as float64 (exact below 2^53 patches).
 */
#ifndef DDCCA_H
#define DDCCA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DDCCA_API __attribute__((visibility("default")))
#else
#define DDCCA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DDCCA_OK = 0,
  DDCCA_ESHAPE = 1,
  DDCCA_ECONFIG = 2,
  DDCCA_ENUMERICAL = 3,
  DDCCA_ECUDA = 4
};

/* Library ABI version (bumped on any signature change). */
DDCCA_API int ddcca_version(void);

/* Thread-local message of the last failing call on this thread. */
DDCCA_API const char* ddcca_last_error(void);

/* Length in float64 of one moment payload for (dim, class_count). */
DDCCA_API int64_t ddcca_payload_len(int dim, int class_count);

/* Geometry shared by the patch-based kernels; restates PatchGeometry
 * (patches.py:22-65): zero_same pads top=(l1-1)//2, left=(l2-1)//2, output
 * grid ceil(p/stride) x ceil(q/stride); padding "none" has no pads. */
typedef struct {
  int p, q;            /* map height, width */
  int l1, l2;          /* window height, width */
  int stride;          /* >= 1 */
  int zero_same;       /* 1 = "zero_same", 0 = "none" */
} ddcca_geom;

/* ---------------------------------------------------------------------
 * K1+K2+K3 — per-batch partial moments
 * Replaces: cascade._batch_accumulator_job / accumulate_layer_moments
 *           (cascade.py:155-189) including extract_patch_stack
 *           (patches.py:97-125) and accumulate_batch (moments.py:86-110).
 * maps1/maps2: (n_maps, p, q) float32, view 1 / view 2, maps of one sample
 *   contiguous, samples in manifest order.
 * map_label: (n_maps,) int32 class of each map, in [0, class_count).
 * batch_offsets_host: HOST array (n_batches+1) of map offsets; batch b is
 *   maps [off[b], off[b+1]) (the BatchSpec partition, patches.py:148-157).
 * partials: (n_batches, payload_len) float64 output, one accumulator per
 *   batch — the reference's per-batch MomentAccumulator.
 * center: subtract each patch's mean (extract_patch_stack center=True).
 * Stride-1 geometries use the exact windowed-autocorrelation form (float64
 * products of float32 inputs are exact); other strides use explicit
 * float64 patch columns. Deterministic: fixed reduction order.
 * ------------------------------------------------------------------- */
DDCCA_API size_t ddcca_moments_workspace(const ddcca_geom* g, int n_batches, int64_t max_maps_per_batch,
                               int class_count);
DDCCA_API int ddcca_moments_partial(const float* maps1, const float* maps2, const int32_t* map_label,
                          const int64_t* batch_offsets_host, int n_batches, const ddcca_geom* g,
                          int center, int class_count, double* partials, void* ws, size_t ws_bytes,
                          void* stream);

/* Same, with flags. DDCCA_MOMENTS_F32_BLOCKS: the lag products of one map's
 * row slab (<= 48 rows) accumulate in float32 and are added to the float64
 * sums per map (FFMA instead of DFMA; ~1e-7 relative per lag sum instead of
 * exact). Meant for layers whose inputs are filter responses (no DC term);
 * applies to the TMA lag path (q % 4 == 0, 5x5 / 7x7 / 9x9), exact elsewhere. */
#define DDCCA_MOMENTS_F32_BLOCKS 1
/* DDCCA_MOMENTS_FINE_SPLITS: batches of <= 128 maps (one map per sample) are
 * split into 32-map slices instead of one 128-map slice (4x the CTAs of a
 * first layer). Split boundaries never depend on the other batches of the
 * call, so each batch's partial is the same in any call or on any rank. */
#define DDCCA_MOMENTS_FINE_SPLITS 2
DDCCA_API int ddcca_moments_partial_ex(const float* maps1, const float* maps2, const int32_t* map_label,
                             const int64_t* batch_offsets_host, int n_batches, const ddcca_geom* g,
                             int center, int class_count, double* partials, void* ws, size_t ws_bytes,
                             int flags, void* stream);

/* ---------------------------------------------------------------------
 * K9 — fixed left-to-right pairwise tree over n_parts payloads
 * Replaces: pairwise_merge (moments.py:132-144); merge (moments.py:113-129)
 * is the n_parts == 2 case. parts is overwritten (in-place tree); the
 * result is copied to out.
 * ------------------------------------------------------------------- */
DDCCA_API int ddcca_moments_tree(double* parts, int n_parts, int64_t payload_len, double* out, void* stream);

/* ---------------------------------------------------------------------
 * Explicit patch columns (API-level accumulate_batch, moments.py:86-110)
 * x, y: (dim, cols) float64 row-major; labels: (cols,) int64.
 * Adds into payload (in place).
 * ------------------------------------------------------------------- */
DDCCA_API int ddcca_accumulate_columns(const double* x, const double* y, const int64_t* labels, int64_t cols,
                             int dim, int class_count, double* payload, void* stream);

/* ---------------------------------------------------------------------
 * K4+K5 — finalize + DCCA solve on device (finalize over ceil(d*d/1024) CTAs, then
 *         float64 Jacobi: two whitening CTAs in parallel, one solve CTA)
 * Replaces: finalize (moments.py:168-193), solve_dcca (solver.py:216-257),
 *           sym_eig / inv_sqrt (solver.py:90-170), reshape_filters
 *           (solver.py:260-272).
 * payload: one merged accumulator. Outputs (all device, float64 unless
 * noted): fin (5*d*d: c11, c22, cw, cb, ctilde — DiscriminantMoments),
 * w1, w2 (d x count, row-major), rho (count), conv_pack (float32, see
 * ddcca_conv) for both views, status (int32: DDCCA_* code; 0 = ok).
 * payload == NULL: skip finalize and solve from the moments already in
 * `fin` (API-level solve_dcca(DiscriminantMoments, count)).
 * Needs ddcca_solve_workspace(d) bytes of scratch.
 * ------------------------------------------------------------------- */
DDCCA_API size_t ddcca_solve_workspace(int dim);
DDCCA_API int ddcca_solve(const double* payload, int dim, int class_count, double epsilon, int count,
                double* fin, double* w1, double* w2, double* rho, float* conv_pack1, float* conv_pack2,
                int32_t* status, void* ws, size_t ws_bytes, void* stream);

/* finalize only (moments.py:168-193): fin = [c11 | c22 | cw | cb | ctilde]. */
DDCCA_API int ddcca_finalize(const double* payload, int dim, int class_count, double epsilon, double* fin,
                             int32_t* status, void* stream);

/* Sign binarization + LSB-first hash of consecutive groups of n_bits maps
 * (binarize + hash_combine, encoder.py:50-68): maps (n_groups*n_bits, plane)
 * float32 -> codes (n_groups, plane) uint8 (n_bits <= 8) or uint16. */
DDCCA_API int ddcca_sign_hash(const float* maps, int64_t n_groups, int n_bits, int64_t plane, void* codes,
                              void* stream);

/* Standalone symmetric eigensolver (sym_eig, solver.py:90-158) and
 * inverse square root (inv_sqrt, solver.py:161-170) on one n x n matrix.
 * mode 0: w (n), v (n x n); mode 1: r = inv_sqrt(s) into v, w = eigvals. */
DDCCA_API int ddcca_sym_eig(const double* s, int n, int mode, double* w, double* v, int32_t* status, void* ws,
                  size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------
 * K6 — multi-filter convolution with per-window centering
 * Replaces: apply_filters (cascade.py:108-126) / conv2d (cascade.py:93-100).
 * in: (n_maps, p, q) float32. out: (n_maps, count, oh, ow) float32,
 * filter-minor (children of one input map contiguous, cascade.py:123-125).
 * conv_pack: float32 [d][count] weights (tap-major) as written by
 * ddcca_solve or ddcca_pack_filters.
 * ------------------------------------------------------------------- */
DDCCA_API int ddcca_pack_filters(const double* filters, int count, int dim, float* conv_pack, void* stream);
DDCCA_API int ddcca_conv(const float* in, int64_t n_maps, const ddcca_geom* g, const float* conv_pack, int count,
               int center, float* out, void* stream);

/* ---------------------------------------------------------------------
 * K6-final + K7 — last-layer conv fused with sign binarization and the
 * LSB-first 2^count hash (encoder.py:50-68, cascade.py:108-126).
 * codes: (n_maps, oh, ow) uint8 when count <= 8, else uint16.
 * ------------------------------------------------------------------- */
DDCCA_API int ddcca_conv_hash(const float* in, int64_t n_maps, const ddcca_geom* g, const float* conv_pack, int count,
                    int center, void* codes, void* stream);

/* Constant-bank variants (stride 1, square 3/5/7/9 windows, <= 16 filters):
 * the zero-mean taps of each launch are staged into the library's constant
 * tap bank on the launching stream, from HOST memory (the _hw entry points:
 * float32 [d][count], e.g. a host copy of the pack written by ddcca_solve)
 * or straight from the DEVICE pack ddcca_solve wrote (the _dev entry points:
 * no host round trip between the solve and the next layer's conv). The bank
 * is one per device: calls on different streams of one device must be
 * ordered by the caller. ddcca_conv_hist_* runs on the tcgen05 tensor cores
 * (kind::f16, maps and filters scaled by powers of two and split into f16 hi + lo:
 * float32-level responses) when the inputs need no DC shift and the shape is covered
 * (maps of <= 128 rows, q % 4 == 0, <= 8 filters, 3/5/7 windows; DDCCA_CONV_TC=0
 * forces the FFMA kernel). DDCCA_ECONFIG means "shape not covered" (use ddcca_conv /
 * ddcca_conv_hash + ddcca_block_hist). ddcca_conv_hist_hw fuses the last
 * layer's conv, sign hash and non-overlapping block histograms (K6-final +
 * K7 + K8): counts are written as in ddcca_block_hist, n_bits = count.
 * `center` of ddcca_conv_hist_hw: bit 0 = the layer centers its patches
 * (LayerConfig.center); DDCCA_CONV_RESPONSES = the inputs are filter
 * responses of a previous layer (zero-mean), so the float32 shift that keeps
 * image DC out of the sums is skipped (same results within float32 rounding). */
#define DDCCA_CONV_RESPONSES 2
DDCCA_API int ddcca_conv_hw(const float* in, int64_t n_maps, const ddcca_geom* g, const float* conv_pack_host,
                            int count, int center, float* out, void* stream);
DDCCA_API int ddcca_conv_hist_hw(const float* in, int64_t n_maps, const ddcca_geom* g, const float* conv_pack_host,
                                 int count, int center, int block_h, int block_w, void* counts, int count_kind,
                                 int64_t groups_per_row, int64_t row_stride, int64_t group_stride, void* stream);
/* Which kernel the calling thread's last ddcca_conv_hist_* call launched: 1 = tcgen05 tensor
 * cores (f16 two-term split), 0 = FFMA. For roofline accounting. */
DDCCA_API int ddcca_conv_hist_last_path(void);
/* Which kernel the calling thread's last ddcca_conv_hw / ddcca_conv_dev call launched: 1 =
 * tcgen05 tensor cores (same kind::f16 split as the conv-histogram, each map shifted by its mean
 * for centered windows; "same" padding, l1 == l2 in {3, 5, 7}, <= 8 filters, maps of <= 128
 * rows, q % 4 == 0), 0 = FFMA constant-bank kernel. For roofline accounting. */
DDCCA_API int ddcca_conv_last_path(void);
DDCCA_API int ddcca_conv_dev(const float* in, int64_t n_maps, const ddcca_geom* g, const float* conv_pack,
                             int count, int center, float* out, void* stream);
DDCCA_API int ddcca_conv_hist_dev(const float* in, int64_t n_maps, const ddcca_geom* g, const float* conv_pack,
                                  int count, int center, int block_h, int block_w, void* counts, int count_kind,
                                  int64_t groups_per_row, int64_t row_stride, int64_t group_stride, void* stream);

/* ---------------------------------------------------------------------
 * K8 — block histograms of code maps (iq_block_features counts,
 * encoder.py:71-99; block_starts encoder.py:38-44).
 * codes: (n_groups, oh, ow), code_bytes 1 or 2. Output counts for group k
 * at counts + (k / groups_per_row) * row_stride + (k % groups_per_row) *
 * group_stride (elements), laid out [block][bin]. count_kind: 0 = uint8
 * (bpc <= 255), 1 = saturating uint8 (256 <= bpc <= 510: 255 means "255 +
 * remainder of the block"), 2 = uint16.
 * ------------------------------------------------------------------- */
DDCCA_API int ddcca_block_hist(const void* codes, int code_bytes, int64_t n_groups, int oh, int ow, int n_bits,
                     int block_h, int block_w, int step_h, int step_w, void* counts, int count_kind,
                     int64_t groups_per_row, int64_t row_stride, int64_t group_stride, void* stream);

/* Counts -> float64 IQ features through a host-built LUT of bpc+1 values
 * (lut[0] = zero-bin value, lut[k] = -log(k/bpc)), encoder.py:87-97.
 * n_blocks histograms of 2^n_bits bins each, contiguous. */
DDCCA_API int ddcca_iq_expand(const void* counts, int count_kind, int64_t n_blocks, int n_bits, int bpc,
                    const double* lut, double* out, void* stream);

/* ---------------------------------------------------------------------
 * K1 standalone — explicit patch matrix (extract_patch_stack,
 * patches.py:97-125): maps (n_maps, p, q) float64 -> out (dim, n_maps*oh*ow)
 * float64 row-major.
 * ------------------------------------------------------------------- */
DDCCA_API int ddcca_im2col(const double* maps, int64_t n_maps, const ddcca_geom* g, int center, double* out,
                 void* stream);


/* ---------------------------------------------------------------------
 * Downstream nearest-neighbour classifier (classify.py:109-143):
 * pred[i] = label of the training row nearest to query row i, squared
 * euclidean (metric 0, q2 + t2 - 2 q.t, classify.py:113-115) or cosine
 * (metric 1, classify.py:116-120); ties -> lowest label (classify.py:136-138).
 * Rows: row_kind 3 = float64 features; 0 / 2 = u8 / u16 block counts expanded
 * through `lut` (lut_len = bpc + 1 values, the iq LUT) while staged.
 * Saturating-u8 counts go through ddcca_counts_to_u16 first.
 * ------------------------------------------------------------------- */
DDCCA_API size_t ddcca_nn_workspace(int64_t n_query, int64_t n_train);
DDCCA_API int ddcca_nn_classify(const void* query, int64_t n_query, const void* train, int64_t n_train,
                                int64_t dim, int row_kind, const double* lut, int lut_len,
                                const int64_t* train_labels, int metric, int64_t* pred, void* workspace,
                                size_t ws_bytes, void* stream);
/* Linear one-vs-all prediction (ridge models, classify.py:140-142): pred[i] =
 * the class of the largest x_i . w_c + bias_c, lowest class id on ties
 * (class_ids[c] per weight row). Float64 rows; workspace ddcca_nn_workspace(nq, n_class). */
DDCCA_API int ddcca_linear_classify(const double* query, int64_t n_query, const double* weights, int64_t n_class,
                                    int64_t dim, const double* bias, const int64_t* class_ids, int64_t* pred,
                                    void* workspace, size_t ws_bytes, void* stream);
/* Saturating-u8 block counts (count_kind 1) -> exact u16 counts. */
DDCCA_API int ddcca_counts_to_u16(const uint8_t* counts, int64_t n_blocks, int bins, int bpc, uint16_t* out,
                                  void* stream);

/* ---------------------------------------------------------------------
 * Second view (views.py:41-58): 8-neighbour LBP map of each (p, q) float32
 * image, strict neighbour > centre, bits clockwise from the top-left,
 * zero padding, code / 255; out may not alias images.
 * ------------------------------------------------------------------- */
DDCCA_API int ddcca_lbp(const float* images, int64_t n, int p, int q, float* out, void* stream);

/* ---------------------------------------------------------------------
 * Host ingestion (dataset.py:68-118): binary PGM (P5) decode, values /
 * maxval (8-bit, or big-endian 16-bit when maxval > 255), '#' comments in
 * the header. ddcca_pgm_load_many decodes n same-size files in parallel
 * (threads) into out[n][height][width] float32 (pinned host memory works).
 * Host-only: no GPU needed. Errors: DDCCA_ESHAPE + ddcca_last_error().
 * ------------------------------------------------------------------- */
DDCCA_API int ddcca_pgm_info(const char* path, int* width, int* height, int* maxval, int64_t* payload_offset);
DDCCA_API int ddcca_pgm_load_many(const char* const* paths, int64_t n, int height, int width, float* out,
                                  int threads);

/* Feature CSV (run_extract, pipeline.py:143-166) straight from host block
 * counts: row r is "first_index + r,v,v,...\n" with v = lut_str[count]
 * (the caller's format(lut[k], ".17g") strings for k = 0..bpc). Count kinds as
 * ddcca_block_hist; `bins` per block. Host-only, `threads` formatting workers. */
DDCCA_API int ddcca_write_feature_csv(const void* counts, int count_kind, int64_t rows, int64_t cols, int bins,
                                      int bpc, const char* const* lut_str, const int* lut_len,
                                      int64_t first_index, const char* path, int threads);

#ifdef __cplusplus
}
#endif
#endif /* DDCCA_H */
