/*
 * dquant_b200.h -- C ABI of the B200-native DecoQuant hot path.
 *
 * Plain pointers and sizes only: every tensor argument is a DEVICE pointer
 * (cudaMalloc / torch CUDA storage) unless its name starts with h_, every
 * `stream` is a cudaStream_t passed as void*.  Calls are stream-ordered and
 * never allocate: scratch comes from a caller-owned workspace whose size the
 * matching *_workspace_size query returns.  No global mutable state beyond a
 * thread-local error string.
 *
 * Status: every entry point returns DQ_OK (0) or a DQ_ERR_* code; the message
 * is in dq_last_error().  Errors that depend on DEVICE data (non-finite input,
 * out-of-range codes) are reported through a caller-provided device int32
 * `flags` word (DQ_FLAG_* bits), which the host reads after the stream is
 * synchronised -- this keeps the hot path free of host round trips.
 *
 * Reference interface replaced (the reference is pure Python; its "operator
 * API" is the dquant module surface, /root/reference/pkg/src/dquant/__init__.py:10-77):
 *   dq_plan_shapes ................ mpo.plan_shapes            mpo.py:73-96
 *   dq_pack / dq_unpack ............ quantize.pack/unpack/unpack_range  quantize.py:66-120
 *   dq_quantize_rtn ................ quantize.quantize_rtn      quantize.py:123-151
 *   dq_quantize_rtn_f64 ............ quantize.quantize_rtn on float64 input (quantize.py:144 multiplies in f64)
 *   dq_dequantize .................. quantize.dequantize        quantize.py:154-157
 *   dq_decompose_batched ........... mpo.decompose (n=2)        mpo.py:153-178
 *   dq_sym_eig_batched ............. the SVDs of mpo.decompose for n > 2 (per TT stage, Gram form)
 *   dq_deco_quantize_batched ....... compress.deco_quantize     compress.py:85-94
 *   dq_deco_quantize_asym_batched .. (opt-in per-channel asymmetric mode of north_star; no
 *                                    reference counterpart, parity against the oracle only)
 *   dq_deco_dequantize_batched ..... compress.deco_dequantize + mpo.reconstruct
 *                                                              compress.py:105-107, mpo.py:181-198
 *   dq_fused_matmul_t .............. compress.fused_matmul_t    compress.py:195-231
 *   dq_fused_matmul ................ compress.fused_matmul      compress.py:159-192
 *   dq_relayout .................... QuantizedTensor.payload wire order  quantize.py:11-14
 *   dq_decode_attention ............ KvCache.attention_scores + softmax + per-segment
 *                                    fused_matmul (kvcache.py:188-217, compress.py:159-192)
 *   dq_tail_append ................. LayerCache.append (tail write)  kvcache.py:116-123
 */
#ifndef DQUANT_B200_H
#define DQUANT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirrors dquant/errors.py:4-61 class names) ---------- */
#define DQ_OK 0
#define DQ_ERR_UNSUPPORTED_BITS 1 /* UnsupportedBits   errors.py:28 */
#define DQ_ERR_SHAPE_MISMATCH 2   /* ShapeMismatch     errors.py:8  */
#define DQ_ERR_CORRUPT_PAYLOAD 3  /* CorruptPayload    errors.py:36 */
#define DQ_ERR_NONFINITE 4        /* NonFiniteInput    errors.py:24 */
#define DQ_ERR_RANGE_OVERFLOW 5   /* RangeOverflow     errors.py:32 */
#define DQ_ERR_INVALID_ARG 6      /* bad pointer / size / workspace */
#define DQ_ERR_CUDA 7             /* CUDA runtime error (message has details) */
#define DQ_ERR_UNSUPPORTED 8      /* valid request outside this build's kernels */

/* ---- device-side flag bits written into the caller's `flags` word ------ */
#define DQ_FLAG_NONFINITE 1u
#define DQ_FLAG_RANGE_OVERFLOW 2u
#define DQ_FLAG_JACOBI_NOCONV 4u

/* ---- dtypes ------------------------------------------------------------ */
#define DQ_F32 0
#define DQ_F16 1

/* ---- packed large-core layouts ------------------------------------------
 * DQ_LAYOUT_REF  : the reference wire order, codes of core1 (r, i2, j2) in
 *                  row-major order, payload_size(r*i2*j2, bits) bytes
 *                  (quantize.py:11-14, 66-82).
 * Device layouts (what the fused attention kernel streams; i2p = i2 rounded up to
 * a multiple of 64, bt = b / 64 is a 64-row tile, padding codes encode 0; codes
 * are stored in excess-2^(bits-1) form, i.e. code + 2^(bits-1) unsigned):
 * DQ_LAYOUT_KTILE: (bt, r, 64, j2) with the 64 rows of a tile XOR-swizzled,
 *                  row b' = (b % 64) ^ ((r & 3) * 16 / bits).  One (tile, r-range)
 *                  is one contiguous bulk copy for the QK^T contraction.
 * DQ_LAYOUT_VTILE: (bt, r, j2, 64): the b index innermost, so the PV contraction
 *                  streams codes along its reduction axis.
 * Both need j2*bits % 8 == 0.  dq_relayout converts to/from DQ_LAYOUT_REF.
 */
#define DQ_LAYOUT_REF 0
#define DQ_LAYOUT_KTILE 1
#define DQ_LAYOUT_VTILE 2

/* ---- n=2 plan (mpo.py:73-96 with n=2; r = bond, mpo.py:54-63) ---------- */
typedef struct dq_plan2 {
  int64_t i1, i2, j1, j2, r;
} dq_plan2;

const char* dq_last_error(void);
int dq_version(void);

/* host-only: general n (i_factors/j_factors hold n entries each) */
int dq_plan_shapes(int64_t rows, int64_t cols, int32_t n, int64_t* h_i_factors, int64_t* h_j_factors);
int dq_make_plan2(int64_t rows, int64_t cols, dq_plan2* h_plan);
/* bytes of one packed large core in `layout` (host-only) */
int dq_layout_bytes(const dq_plan2* h_plan, int32_t bits, int32_t layout, int64_t* h_bytes);

/* ---- K1 codec ---------------------------------------------------------- */
int dq_pack(const int8_t* codes, int64_t count, int32_t bits, uint8_t* payload, int32_t* flags, void* stream);
int dq_unpack(const uint8_t* payload, int64_t payload_bytes, int64_t start, int64_t count, int32_t bits,
              int8_t* codes, void* stream);

/* ---- K2 quantizer: one symmetric scale per tensor ---------------------- */
int dq_quantize_workspace_size(int64_t count, size_t* h_bytes);
int dq_quantize_rtn(const float* t, int64_t count, int32_t bits, float* scale, uint8_t* payload, int32_t* flags,
                    void* workspace, size_t workspace_bytes, void* stream);
/* float64 input: amax and t*qmax/amax on the original f64 values, bit-exact with the reference */
int dq_quantize_rtn_f64(const double* t, int64_t count, int32_t bits, float* scale, uint8_t* payload, int32_t* flags,
                        void* workspace, size_t workspace_bytes, void* stream);
int dq_dequantize(const uint8_t* payload, int64_t count, int32_t bits, const float* scale, float* out, void* stream);

/* ---- K3 write path: batched n=2 TT-SVD (+ quantize) -------------------
 * blocks: nblk matrices of rows x cols (row-major, dtype in_dtype), contiguous.
 * core0 : nblk x (i1*j1*r) f32 (shape (1,i1,j1,r) each)
 * core1 : nblk x (r*i2*j2) f32 (shape (r,i2,j2,1) each)
 * payload: nblk packed cores, block k at payload + k*payload_stride, in `layout`
 * scale : nblk f32
 */
int dq_decompose_workspace_size(int64_t nblk, int64_t rows, int64_t cols, size_t* h_bytes);
int dq_decompose_batched(const void* blocks, int32_t in_dtype, int64_t nblk, int64_t rows, int64_t cols,
                         float* core0, float* core1, int32_t* flags, void* workspace, size_t workspace_bytes,
                         void* stream);
/* K3's eigensolver alone (Householder + implicit QL, fp64): nblk symmetric n x n matrices (n <= 64),
 * gram [nblk][64][64] (upper triangle read, row stride 64) -> vectors [nblk][64][64] (column k =
 * eigenvector k, largest-|entry| positive) and values [nblk][64] in descending order; no convergence
 * -> DQ_FLAG_JACOBI_NOCONV in *flags.  The TT-SVD stages of chains longer than 2 (mpo.py:153-178)
 * are Gram -> this -> projection. */
int dq_sym_eig_batched(const double* gram, int64_t nblk, int32_t n, double* vectors, double* values, int32_t* flags,
                       void* stream);
/* same as dq_decompose_batched with an explicit n=2 plan (any split whose bond r <= 64) */
int dq_decompose_plan_batched(const void* blocks, int32_t in_dtype, int64_t nblk, const dq_plan2* h_plan,
                              float* core0, float* core1, int32_t* flags, void* workspace, size_t workspace_bytes,
                              void* stream);
int dq_deco_quantize_batched(const void* blocks, int32_t in_dtype, int64_t nblk, int64_t rows, int64_t cols,
                             int32_t bits, int32_t layout, float* core0, uint8_t* payload, int64_t payload_stride,
                             float* scale, int32_t* flags, void* workspace, size_t workspace_bytes, void* stream);
/* Opt-in per-channel ASYMMETRIC quantisation of core1 (north_star; not in the reference, whose
 * quantizer is per-tensor symmetric, quantize.py:123-151 -- parity unpinned, checked against the
 * oracle's restatement only).  Channel = (r, e) over b, bits in {2, 4}, qmu = 2^bits - 1:
 *   s = f32((max - min) / qmu)   (|max| or 1 for a constant channel)
 *   z = clip(floor(-min / s + 0.5), 0, qmu),  u = clip(floor(v / s + 0.5) + z, 0, qmu)   (fp64)
 *   value = s * (u - z);  the raw codes u are packed in `layout` (KTILE / VTILE / REF).
 * channels: nblk x [2][r][j2] f32 (the scales s, then the zero points z as floats). */
int dq_deco_quantize_asym_batched(const void* blocks, int32_t in_dtype, int64_t nblk, int64_t rows, int64_t cols,
                                  int32_t bits, int32_t layout, float* core0, uint8_t* payload,
                                  int64_t payload_stride, float* channels, int32_t* flags, void* workspace,
                                  size_t workspace_bytes, void* stream);
/* copy of core0 (fp16 or fp32) in the attention-friendly layout out[a][r][c] (i1 x r x j1),
 * normalised by a power of two per block so that max|out| is in [0.5, 1); norm[blk] receives
 * that factor (core0 = out * norm).  norm may be null (then no normalisation). */
int dq_core0_relayout(const float* core0, int64_t nblk, const dq_plan2* h_plan, void* out, int32_t out_dtype,
                      float* norm, void* stream);

/* ---- K4 reconstruct (dequant + contraction), batched ------------------- */
int dq_deco_dequantize_batched(const float* core0, const uint8_t* payload, int64_t payload_stride, int32_t layout,
                               const float* scale, int64_t nblk, int64_t rows, int64_t cols, int32_t bits,
                               void* out, int32_t out_dtype, void* stream);

/* layout conversion of packed cores (e.g. device layouts -> reference wire order) */
int dq_relayout(const uint8_t* src, int32_t src_layout, int64_t src_stride, uint8_t* dst, int32_t dst_layout,
                int64_t dst_stride, int64_t nblk, const dq_plan2* h_plan, int32_t bits, void* stream);

/* ---- generic fused reads (any n=2 plan with i1*j1 <= 64) -----------------
 * x: p x cols (f32) -> out: p x rows (f32) = x @ W^T
 * x: p x rows (f32) -> out: p x cols (f32) = x @ W
 * meter (optional, device uint64[2], WorkingSetMeter compress.py:23-33): the kernels add their own
 * measurement -- [0] = max dequantized codes one CTA holds at once, [1] += codes dequantized.
 */
int dq_fused_matmul_t(const float* x, int64_t p, const float* core0, const uint8_t* payload, int32_t layout,
                      const float* scale, int64_t rows, int64_t cols, int32_t bits, float* out, uint64_t* meter,
                      void* stream);
int dq_fused_matmul(const float* x, int64_t p, const float* core0, const uint8_t* payload, int32_t layout,
                    const float* scale, int64_t rows, int64_t cols, int32_t bits, float* out, uint64_t* meter,
                    void* stream);

/* ---- K5 fused dequant + decode attention (D = 128, j = (8,16)) -----------
 * One "unit" is one (sequence, kv head) of one layer; g query heads attend to it.
 * A unit owns zero or more compressed segments (prefill segment, sealed chunks)
 * and an fp16 tail.  Segment s of the work list belongs to unit seg_unit[s].
 */
typedef struct dq_segment {
  const uint8_t* k_codes; /* DQ_LAYOUT_KTILE */
  const uint8_t* v_codes; /* DQ_LAYOUT_VTILE */
  const float* k_g0;      /* fp32 [i1][r][8]  (dq_core0_relayout, normalised): score side */
  const void* v_g0;       /* [i1][r][8] (dq_core0_relayout, normalised): output side; fp32, or fp16 where
                             dq_attention_g0v_dtype says so */
  float k_scale, v_scale; /* quantizer scale times the G0 normalisation factor */
  int32_t T;          /* tokens in the segment */
  int32_t i1, i2, r;  /* plan of (T,128) */
  int32_t i2p;        /* padded i2 of the device layouts */
  int32_t unit;       /* owning unit */
  int32_t token0;     /* first token index of the segment inside its unit */
  int32_t pad_;
  const float* k_ch;  /* asymmetric mode: [2][r][16] per-channel scales and zero points (see
                         dq_deco_quantize_asym_batched); k_scale / v_scale then carry only the G0
                         normalisation.  Null: the reference's symmetric per-tensor codes */
  const float* v_ch;
} dq_segment;

typedef struct dq_attn_args {
  const uint16_t* q;      /* fp16 [units][g][128] (units = virtual units, see head_groups) */
  uint16_t* out;          /* fp16 [units][g][128] (bf16 with out_bf16) */
  const dq_segment* segs; /* device array [nseg] */
  int32_t nseg;
  int32_t units;
  int32_t g;              /* query heads per kv head (1..8) */
  int32_t bits;           /* 2, 4 or 8 */
  uint16_t* tail_k;       /* fp16 [units][tail_cap][128] (may be null if tail_len==0 and no append) */
  uint16_t* tail_v;
  int32_t* tail_len;      /* device [units] */
  int32_t tail_cap;
  int32_t chunk_b;        /* max b rows per work item (sub-item) of the split kernel: 256 */
  float sm_scale;         /* softmax scale, 1/sqrt(128) for the reference scores */
  /* work list (built by dq_attention_plan) */
  const int32_t* work;    /* device int32 [nwork][3] = (segment, b0, 64-row tiles) */
  int32_t nwork;
  int32_t max_parts;      /* partial slots per unit (>= work items of any unit + 1) */
  const int32_t* unit_part0; /* device [units]: first partial slot of each unit */
  const int32_t* work_part;  /* device [nwork]: partial slot of each work item */
  const int32_t* unit_nparts;/* device [units] */
  int32_t* sched;            /* device [2] scheduler counters, zero before the first launch (self-resetting) */
  float* part_o;          /* workspace [total_parts][g][128] f32 */
  float* part_ml;         /* workspace [total_parts][g][2]   f32 (max, sum) */
  int32_t phases;         /* bit 0: split kernel, bit 1: combine kernel, bit 2: prepare kernel; 0: all;
                             bit 3: launch the split kernel without its PDL edge (timing) */
  int32_t nctas;          /* persistent split-kernel CTAs (dq_attention_ctas); <= 0 or >= nwork: one per item */
  int64_t* trace;         /* optional (profiling): [nwork][8] global-timer stamps per work item */
  void* wimg;             /* workspace [nseg][wimg_stride]: per-segment W images (prepare kernel) */
  int64_t wimg_stride;    /* >= dq_attention_wimg_bytes(g) */
  const uint16_t* app_k;  /* optional fp16 [units / head_groups][128]: appended to the tail AFTER */
  const uint16_t* app_v;  /*   the attention (the combine kernel does dq_tail_append's work) */
  int32_t head_groups;    /* GQA groups wider than the kernels' g: a kv head's g_total = g * head_groups
                             query heads run as head_groups "virtual units" u * head_groups + k (each g
                             heads, same codes; segs/q/out/partials indexed by virtual unit, the tail and
                             the combine grid by kv head u).  0 or 1: none */
  int32_t path;           /* split kernel: 0 = mma.sync (all plans), 1 = tcgen05 (int4, g = 1, r = 64, i1 = 8),
                             2 = tcgen05 GQA (int4, g = 8, r = 64, i1 = 8) */
  int32_t asym;           /* 1: every segment is in the asymmetric per-channel mode (path 0, 2- / 4-bit) */
  int32_t out_bf16;       /* 1: out is bf16 [units][g][128] instead of fp16 (read directly by a model's bf16
                             projections; the merged fp32 value is rounded once) */
} dq_attn_args;

/* bytes of one per-segment W image (the wimg stride) for a GQA group of g heads */
int dq_attention_wimg_bytes(int32_t g, int64_t* h_bytes);

/* element type (DQ_F16 / DQ_F32) of the dq_segment.v_g0 tables the split kernel of (g, path, asym,
 * chunk_b) reads: fp16 where it computes the W image itself (path 0, g = 1, symmetric, items of
 * <= 256 rows: no prepare kernel) */
int dq_attention_g0v_dtype(int32_t g, int32_t path, int32_t asym, int32_t chunk_b, int32_t* h_dtype);

/* resident split-kernel CTAs on the current device (SMs x CTAs per SM): the persistent grid */
int dq_attention_ctas(int32_t g, int32_t bits, int32_t* h_ctas);

/* host helper: fill the work/partial tables (host arrays) for a host copy of the segment
 * table: every segment is cut into ceil(tiles / (chunk_b / 64)) near-equal work items of
 * 64-row b tiles.  h_work [max_work][3] may be null (count only). */
int dq_attention_plan(const dq_segment* h_segs, int32_t nseg, int32_t units, int32_t chunk_b, int32_t max_work,
                      int32_t* h_work, int32_t* h_nwork, int32_t* h_work_part, int32_t* h_unit_part0,
                      int32_t* h_unit_nparts, int32_t* h_total_parts);
int dq_decode_attention(const dq_attn_args* h_args, void* stream);

/* append one token row per unit into the fp16 tail (kvcache.py:116-123) */
int dq_tail_append(const uint16_t* k_rows, const uint16_t* v_rows, int32_t units, uint16_t* tail_k,
                   uint16_t* tail_v, int32_t* tail_len, int32_t tail_cap, void* stream);

/* ---- decode-harness kernels (no reference counterpart: the reference
 * has no model, its toy analogue is kvcache.py:234-309).  The elementwise work around the
 * cuBLAS projections of model.py's LLaMA-shaped decoder; all tensors bf16 (uint16_t) unless
 * stated, row-major, device pointers. */
/* x_out = x + y (skipped when y is NULL: x is the residual as is), h = RMSNorm(x_out) * w */
int dq_model_add_rmsnorm(const uint16_t* x, const uint16_t* y, const uint16_t* w, uint16_t* x_out, uint16_t* h,
                         int32_t rows, int32_t hidden, float eps, void* stream);
/* fused QKV rows (batch, (heads + 2 kv_heads) * 128) -> rotary q (batch, heads, 128) fp16,
 * rotary k and plain v (batch, kv_heads, 128) fp16, at decode position *pos (device int64) */
int dq_model_qkv_rope(const uint16_t* qkv, int32_t batch, int32_t heads, int32_t kv_heads, const int64_t* pos,
                      float theta, uint16_t* q, uint16_t* k, uint16_t* v, void* stream);
/* SwiGLU: gate_up rows (rows, 2 ffn) = [gate | up] -> out (rows, ffn) = silu(gate) * up */
int dq_model_silu_mul(const uint16_t* gate_up, int32_t rows, int32_t ffn, uint16_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DQUANT_B200_H */
