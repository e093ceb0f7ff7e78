/*
 * blockmm_b200.h -- C ABI of the B200-native randomized block matrix
 * multiplication hot path (arXiv 2105.04940).
 *
 * The reference (/root/reference/pkg/src/blockmm) is pure Python/NumPy and has
 * no FFI layer; its drop-in boundary is the Python API re-exported from
 * pkg/src/blockmm/__init__.py:10-99.  Each entry point below replaces the
 * NumPy/BLAS computation inside one reference function (cited per entry);
 * the Python package paper_2105_04940_b200 binds them with ctypes and keeps
 * the reference's names, arguments, return types and ValueError behaviour.
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless named host_*;
 *   - matrices are row-major with an explicit leading dimension (elements);
 *   - batched entry points take `batch` problems of identical shape, problem
 *     b starting at base + b * stride (elements);
 *   - `stream` is a cudaStream_t passed as void*; all work is enqueued on it
 *     and nothing synchronises the host unless stated;
 *   - returns BMM_OK (0) or a negative BMM_E_* code; bmm_last_error() gives a
 *     thread-local message for the last failure.
 *   - per-problem validation outcomes that the reference reports as
 *     ValueError/AssertionError are written to a device `status` array (see
 *     BMM_ST_*), because they depend on device-computed values.
 */
#ifndef BLOCKMM_B200_H
#define BLOCKMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types */
#define BMM_F64 0
#define BMM_F32 1

/* return codes */
#define BMM_OK 0
#define BMM_E_ARG (-1)
#define BMM_E_CUDA (-2)
#define BMM_E_UNSUPPORTED (-3)

/* per-problem device status codes (reference error it stands for) */
#define BMM_ST_OK 0
#define BMM_ST_ZERO_SCORE 1        /* plan.py:390-391,410-411,453-454 "all blocks have zero score" */
#define BMM_ST_CAUCHY_SCHWARZ 2    /* plan.py:119-120 BlockScores check                             */
#define BMM_ST_RADICAND 3          /* plan.py:358-360 radicand negative beyond slack               */
#define BMM_ST_ALL_ZERO_WEIGHT 4   /* plan.py:267-268 "all weights are zero"                        */
#define BMM_ST_BAD_WEIGHT 5        /* plan.py:265-266 weights must be finite and >= 0              */
#define BMM_ST_CAP_BELOW_FLOOR 6   /* plan.py:285-286                                               */
#define BMM_ST_BELOW_FLOORS 7      /* plan.py:287-288 (diag = number of floors)                     */
#define BMM_ST_ABOVE_CAPS 8        /* plan.py:289-290 (diag = total caps)                           */
#define BMM_ST_NO_CONVERGE 9       /* plan.py:306,321,347 AssertionError                            */
#define BMM_ST_NOT_PLACED 10       /* plan.py:342 AssertionError                                    */
#define BMM_ST_EMPTY_SUPPORT 11    /* estimators.py:39-40                                           */
#define BMM_ST_PLAN_MISMATCH 12    /* plan.py:146-152 zero budget on a scored block (diag = block)  */
#define BMM_ST_BAD_PROBS 13        /* plan.py:68-69 non-finite probabilities (NaN/Inf input; diag = block) */

/* budget rules for bmm_budgets (plan.py allocators) */
#define BMM_RULE_EXPLICIT 0   /* integerize(weights, c, caps, floor)          plan.py:242-347 */
#define BMM_RULE_ONC 1        /* allocate_by_score_sums: w = s                plan.py:403-413 */
#define BMM_RULE_OPL 2        /* allocate_optimal: w = sqrt(max(s^2-g^2,0))   plan.py:383-400 */
#define BMM_RULE_TWO_STEP 3   /* allocate_two_step: w = sqrt(|s^2-pilot^2|)   plan.py:465-470 */
#define BMM_RULE_UU 4         /* allocate_uniform: w = 1, floor all           plan.py:416-421 */
#define BMM_RULE_PILOT 5      /* two-step pilot: c draws per block with p0 != 0 (s > 0, or every
                                 block when s is NULL)        plan.py:447,457-460 */

/* ---------------------------------------------------------------- library */
int bmm_version(void);
const char* bmm_last_error(void);
/* number of kernels this library has launched since load (evidence counter) */
int64_t bmm_launch_count(void);

/* Strided copy (cudaMemcpy2DAsync; kind 1 = host->device, 2 = device->host,
 * 3 = device->device), graph-capturable: the streamed end-to-end path copies
 * block-column slabs of a pinned host M so work on early blocks overlaps the
 * transfer of later ones.                                                    */
int bmm_copy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes,
               int64_t height, int kind, void* stream);

/* ---------------------------------------------------------------- K1 norms
 * colsq[b, i] = sum_h M[b][h, i]^2, accumulated sequentially over h in float64
 * (numpy's order for np.linalg.norm(M, axis=0) on a C-ordered matrix,
 * matrix.py:107-109).  With accumulate != 0 the chain continues from the
 * values already in colsq (exact row-slab chunking).
 * rowsq[b, i] = numpy-pairwise sum over f of N[b][i, f]^2 in float64
 * (np.linalg.norm(N, axis=1), matrix.py:112-114).
 * Either side may be skipped by passing a NULL matrix pointer.
 * float32 inputs are upcast element-wise (exact squares), which equals the
 * reference run on the float64-upcast matrices.                            */
int bmm_norms(int dtype,
              const void* M, int64_t m, int64_t n, int64_t ldm, int64_t strideM,
              const void* N, int64_t p, int64_t ldn, int64_t strideN,
              int64_t batch, int accumulate,
              double* colsq, double* rowsq, void* stream);

/* ---------------------------------------------------------------- K2 plan
 * Per block k (offsets[0..K], shared by all problems):
 *   sc[i]   = sqrt(colsq[i]) * sqrt(rowsq[i])                     plan.py:165-167
 *   probs   = optimal_probabilities: sc/pw(sc) then p/pw(p),
 *             all-zero vector for a zero-score block              plan.py:192-206
 *   s[k]    = sc[o] + pw(sc[o+1:e])  (np.add.reduceat)            plan.py:170-173
 *   fnorm[k]= ||M^k||_F * ||N_k||_F (SSM block weights)            plan.py:483-492
 *   cum/last: optional fused inverse-CDF tables of probs (see bmm_block_cdf)
 * probs / s / fnorm / cum may be NULL to skip.  colsq/rowsq/probs/cum stride
 * = n, s/fnorm/last stride = K.  One warp per block; max_len >= the largest
 * block size (blocks up to 5120 elements are processed in shared memory).  */
int bmm_block_probs(const double* colsq, const double* rowsq, int64_t n,
                    const int64_t* offsets, int64_t K, int64_t batch, int64_t max_len,
                    double* probs, double* s, double* fnorm,
                    double* cum, int64_t* last_support, void* stream);

/* SSM block probabilities q = f / pw(f) (plan.py:493-496); status gets
 * BMM_ST_ZERO_SCORE when pw(f) == 0.                                        */
int bmm_normalize(const double* f, int64_t K, int64_t batch, double* q,
                  int32_t* status, void* stream);

/* Integer budgets (plan.py:242-347 integerize, with the weights/caps/floors
 * of the allocator named by `rule`).
 *   s      : score sums (K per problem; unused for UU / EXPLICIT)
 *   aux    : squared norms g_k^2 (OPL) / pilot^2 (TWO_STEP), as the segmented
 *            square-sum GEMM returns them (the kernel takes sqrt and squares
 *            again, the reference's rounding path); weights (EXPLICIT)
 *   sizes  : block sizes n_k (K, shared)
 *   caps   : EXPLICIT only, optional explicit caps (K per problem) or NULL
 *   floors : EXPLICIT only, optional uint8 floor mask (K per problem) or NULL
 *   c      : budget per problem (batch entries)
 *   cap    : allocator `cap` flag
 *   budgets: out, int64 K per problem;  col_off: out, K+1 per problem (may be NULL)
 *   status, diag: out, one per problem;  notes: out, 1 if the weights fell
 *            back to the score sums (plan.py:394-398, 467-469)
 *   ws     : workspace of bmm_budgets_workspace(K) bytes per problem        */
int64_t bmm_budgets_workspace(int64_t K);
int bmm_budgets(int rule, const double* s, const double* aux, const int64_t* sizes,
                const int64_t* caps, const uint8_t* floors,
                int64_t K, int64_t batch, const int64_t* c, int cap,
                int64_t* budgets, int64_t* col_off, int32_t* status, int64_t* diag,
                int32_t* notes, void* ws, void* stream);

/* ---------------------------------------------------------------- K3 sampler
 * Per-block inverse-CDF tables: cum = np.cumsum(p) (sequential) and the last
 * index with p > 0 (estimators.py:37-38).  len = offsets[K] per problem.     */
int bmm_block_cdf(const double* probs, const int64_t* offsets, int64_t K, int64_t batch,
                  int64_t n, double* cum, int64_t* last_support, void* stream);

/* numpy SeedSequence -> PCG64 seeding of child streams:
 *   child j of problem b is SeedSequence(entropy, spawn_key = key + (first_child[b]+j,))
 * words[b, 0..n_words) holds the uint32 assembled entropy *before* the child
 * index (run entropy zero-padded to >= 4 words, then the parent spawn key
 * words).  states[b, j] = {state_hi, state_lo, inc_hi, inc_lo}.
 * Replaces rng.spawn(K) at estimators.py:141,207 and plan.py:456.            */
int bmm_seed_streams(const uint32_t* words, int64_t n_words, const int64_t* first_child,
                     int64_t count, int64_t batch, uint64_t* states, void* stream);

/* Draw budgets[k] indices per block from child stream k (estimators.py:34-44,
 * 77-78): u = (next64 >> 11) * 2^-53, idx = min(upper_bound(cum, u), last),
 * scale = 1/sqrt(c_k * p[idx]).  Outputs are indexed by the global sketch
 * column t = col_off[k] + draw:  column[t] = offsets[k] + idx (global inner
 * index), prob[t] = p[idx], scale[t].  W = col_off[K] per problem; outputs
 * have stride w_stride.  `states` has one stream per block (stride K).
 * max_len >= the largest block size: the block's CDF is staged in shared
 * memory for the binary searches when it fits.
 * The SSM baseline (estimators.py:242-243) is the same call with one block
 * spanning the K block probabilities and the caller's own PCG64 state.    */
int bmm_sample(const double* probs, const double* cum, const int64_t* last_support,
               const int64_t* offsets, int64_t K, int64_t batch, int64_t n, int64_t max_len,
               const int64_t* budgets, const int64_t* col_off, int64_t w_stride,
               const uint64_t* states, int64_t* column, double* prob, double* scale,
               void* stream);

/* Monte Carlo replications of ONE plan (analysis.py:343-366 coverage_check,
 * :390-416 normality_diagnostic; bench.py:258-278 rep loop): as bmm_sample,
 * but probs/cum/last_support/budgets/col_off describe a single problem shared
 * by all `reps` replications; states (reps x K streams) and the outputs
 * (stride w_stride) are per replication.                                    */
int bmm_sample_reps(const double* probs, const double* cum, const int64_t* last_support,
                    const int64_t* offsets, int64_t K, int64_t reps, int64_t n, int64_t max_len,
                    const int64_t* budgets, const int64_t* col_off, int64_t w_stride,
                    const uint64_t* states, int64_t* column, double* prob, double* scale,
                    void* stream);

/* Compressed sketch (K4 prologue): the draws of one column share its scale
 * s_i = 1/sqrt(c_k p_i), so c_i duplicates contribute c_i s_i^2 M[:,i] N[i,:]
 * to C @ D (estimators.py:78-80,175).  Writes the distinct drawn columns in
 * column order to out_column[0..count) with out_scale = s_i sqrt(c_i), zero
 * padding up to min(W, ceil32(count)), and count per problem in out_count.  Gathering and
 * contracting (bmm_gemm_f64_dk) the compressed sketch gives C @ D up to
 * rounding with one rank-1 term per distinct column.  Deterministic.
 * Workspace bmm_compress_workspace(n, batch) bytes.                          */
int64_t bmm_compress_workspace(int64_t n, int64_t batch);
int bmm_compress_sketch(const int64_t* column, const double* scale, int64_t W, int64_t w_stride,
                        int64_t n, int64_t batch, void* ws, int64_t ws_bytes,
                        int64_t* out_column, double* out_scale, int64_t* out_count, void* stream);

/* ---------------------------------------------------------------- K4 gather
 * C[h, t] = M[h, column[t]] * scale[t]        (m x W, ldc)     estimators.py:79
 * D[t, f] = N[column[t], f] * scale[t]        (W x p, ldd)     estimators.py:80
 * The product is formed in float64 and rounded once to out_dtype: with
 * float64 output this is bit-identical to NumPy on float64 (or upcast float32)
 * inputs.
 * Either side may be skipped with a NULL output.                            */
int bmm_gather(int dtype, int out_dtype,
               const void* M, int64_t ldm, int64_t strideM,
               const void* N, int64_t ldn, int64_t strideN,
               int64_t m, int64_t p, const int64_t* column, const double* scale,
               int64_t W, int64_t w_stride, int64_t batch,
               void* C, int64_t ldc, int64_t strideC,
               void* D, int64_t ldd, int64_t strideD, void* stream);
/* bmm_gather for a compressed sketch: only sketch columns t < w_dev[b]
 * (device count from bmm_compress_sketch) are written.                      */
int bmm_gather_dk(int dtype, int out_dtype,
                  const void* M, int64_t ldm, int64_t strideM,
                  const void* N, int64_t ldn, int64_t strideN,
                  int64_t m, int64_t p, const int64_t* column, const double* scale,
                  int64_t W, int64_t w_stride, const int64_t* w_dev, int64_t batch,
                  void* C, int64_t ldc, int64_t strideC, void* D, int64_t ldd, int64_t strideD,
                  void* stream);

/* SSM whole-block gather (estimators.py:244-249): draw t copies block
 * blocks[t] scaled by scale[t]; the sketch columns of draw t start at
 * sk_off[t] (prefix of the drawn widths).                                   */
int bmm_gather_blocks(int dtype,
                      const void* M, int64_t ldm, const void* N, int64_t ldn,
                      int64_t m, int64_t p, const int64_t* offsets,
                      const int64_t* blocks, const double* scale, const int64_t* sk_off,
                      int64_t draws, int64_t W,
                      void* C, int64_t ldc, void* D, int64_t ldd, void* stream);

/* SSM draws as sketch columns for the batched pipeline (equal blocks of
 * block_len): column[b*w_stride + t*block_len + j] = offsets[blocks[b*d_stride
 * + t]] + j, col_scale = scale[b*d_stride + t] -- the hstack of scaled whole
 * blocks of estimators.py:244-249, fed to bmm_compress_sketch and the regular
 * gather / contraction kernels.                                             */
int bmm_expand_blocks(const int64_t* blocks, const double* scale, int64_t draws, int64_t d_stride,
                      const int64_t* offsets, int64_t block_len, int64_t batch,
                      int64_t* column, double* col_scale, int64_t w_stride, void* stream);

/* ---------------------------------------------------------------- K5/K8 GEMM fp64
 * out[b] = A[b] (m x k, lda) @ B[b] (k x nc, ldb), float64 on the DMMA
 * tensor pipe (mma.sync m8n8k4 f64), split-K with a fixed-order reduction
 * (deterministic).  Used for C @ D (estimators.py:175,253) and the exact
 * product M @ N (matrix.py:98-104).  ws: bmm_gemm_f64_workspace bytes.    */
int64_t bmm_gemm_f64_workspace(int64_t m, int64_t nc, int64_t k, int64_t batch);
/* Tile configurations of the DMMA kernels (0..6; tools/tune_dmma.py) for
 * bmm_gemm_f64 and bmm_segsq_f64 (defaults 2 and 0).  Changes their workspace
 * sizes; process-global, not thread-safe.                                  */
int bmm_gemm_f64_set_variant(int gemm_variant, int segsq_variant);
int bmm_gemm_f64(const double* A, int64_t lda, int64_t strideA,
                 const double* B, int64_t ldb, int64_t strideB,
                 int64_t m, int64_t nc, int64_t k, int64_t batch,
                 double* out, int64_t ldo, int64_t strideO,
                 void* ws, int64_t ws_bytes, void* stream);

/* Fused gather + contraction (no sketch in memory): out[b] = C[b] @ D[b] with
 * C[:, t] = M[:, column[t]] * scale[t], D[t, :] = N[column[t], :] * scale[t],
 * evaluated as sum_t M[:, col_t] (scale_t^2 N[col_t, :]) on the DMMA pipe: the
 * A tile is gathered with 8-byte copies, B rows of N are copied whole, and the
 * B fragments are scaled by scale_t^2 in registers.  Same workspace as
 * bmm_gemm_f64(m, nc, W, batch).  estimators.py:143-175 without the C, D
 * round trip through HBM.                                                   */
int bmm_gemm_f64_gather(const double* M, int64_t ldm, int64_t strideM,
                        const double* N, int64_t ldn, int64_t strideN,
                        int64_t m, int64_t nc, const int64_t* column, const double* scale,
                        int64_t W, int64_t w_stride, int64_t batch,
                        double* out, int64_t ldo, int64_t strideO,
                        void* ws, int64_t ws_bytes, void* stream);

/* K9, the fused error epilogue (SURVEY.md §8 b2 `err_sq_out_opt`; relative_error,
 * analysis.py:318-325, as coverage_check uses it, analysis.py:343-380): C @ D as bmm_gemm_f64
 * with err_sq[b] = || ref_b - A_b B_b ||_F^2 taken from the accumulator tiles (or the ordered
 * split-K reduction), ref_b = ref + b * strideR (strideR = 0: one exact product for every
 * replication).  out_opt == NULL: the product is never written to HBM.  Deterministic (fixed
 * thread, warp and tile order).                                                            */
int64_t bmm_gemm_f64_err_workspace(int64_t m, int64_t nc, int64_t k, int64_t batch);
int bmm_gemm_f64_err(const double* A, int64_t lda, int64_t strideA, const double* B, int64_t ldb,
                     int64_t strideB, int64_t m, int64_t nc, int64_t k, int64_t batch,
                     const double* ref, int64_t ldr, int64_t strideR, double* out_opt, int64_t ldo,
                     int64_t strideO, double* err_sq, void* ws, int64_t ws_bytes, void* stream);

/* bmm_gemm_f64 with the inner length read from the device (k_dev[b] <= k_max,
 * e.g. bmm_compress_sketch's count): the split-K plan is re-made on the device
 * for the actual length, so a shorter K costs proportionally less.  Workspace:
 * bmm_gemm_f64_workspace(m, nc, k_max, batch).                               */
int bmm_gemm_f64_dk(const double* A, int64_t lda, int64_t strideA,
                    const double* B, int64_t ldb, int64_t strideB,
                    int64_t m, int64_t nc, int64_t k_max, const int64_t* k_dev, int64_t batch,
                    double* out, int64_t ldo, int64_t strideO, void* ws, int64_t ws_bytes, void* stream);

/* Segmented square-sum GEMM: gsq[b, j] = || A[:, seg_j] @ B[seg_j, :] ||_F^2
 * for segments seg_j = [seg[j], seg[j+1]) of the inner dimension.
 * OPL block product norms g_k^2 (plan.py:183-188) with seg = offsets, and
 * two-step pilot norms ||C0 D0||_F^2 (plan.py:457-464) with seg = pilot
 * sketch offsets.  Deterministic (per-tile partials reduced in order).    */
int64_t bmm_segsq_f64_workspace(int64_t m, int64_t nc, int64_t nseg, int64_t batch);
int bmm_segsq_f64(const double* A, int64_t lda, int64_t strideA,
                  const double* B, int64_t ldb, int64_t strideB,
                  int64_t m, int64_t nc, const int64_t* seg, int64_t nseg, int64_t seg_stride,
                  int64_t batch, double* gsq, void* ws, int64_t ws_bytes, void* stream);
/* The same over a sketch gathered on the fly (as bmm_gemm_f64_gather): the
 * two-step pilot norms ||C0_k D0_k||_F^2 straight from M and N (plan.py:457-464). */
int bmm_segsq_f64_gather(const double* M, int64_t ldm, int64_t strideM,
                         const double* N, int64_t ldn, int64_t strideN,
                         int64_t m, int64_t nc, const int64_t* column, const double* scale,
                         int64_t w_stride, const int64_t* seg, int64_t nseg, int64_t seg_stride,
                         int64_t batch, double* gsq, void* ws, int64_t ws_bytes, void* stream);

/* The same segmented square sums on the int8 tensor cores (Ozaki scheme):
 * every value is split exactly into 8 balanced int8 digits under a power-of-two
 * scale per row of A^k / column of B_k (55 bits), the digit-plane products are
 * accumulated exactly in int32 by tcgen05 kind::i8 MMAs (levels t+u <= 7) and
 * recombined in float64 in the epilogue: float64-level accuracy (~1e-16
 * relative) at int8 tensor-core throughput.  plan.py:183-188 (OPL g_k^2).
 * dtype BMM_F64 or BMM_F32 (float32 read directly, exact upcast).  n_inner
 * bounds seg[nseg] - seg[0] (it sizes the digit planes); a segment longer than
 * 32768 or a negative one, or n_inner exceeded, gives NaN for that problem.
 * Deterministic (fixed-order tile and row reductions).                     */
int64_t bmm_segsq_i8_workspace(int64_t m, int64_t nc, int64_t n_inner, int64_t nseg, int64_t batch);
int bmm_segsq_i8(int dtype, const void* A, int64_t lda, int64_t strideA,
                 const void* B, int64_t ldb, int64_t strideB,
                 int64_t m, int64_t nc, int64_t n_inner, const int64_t* seg, int64_t nseg, int64_t seg_stride,
                 int64_t batch, double* gsq, void* ws, int64_t ws_bytes, void* stream);
/* bmm_segsq_i8 with device timing (CUDA events on `stream`, synchronizes):
 * ms[0] = segment prep + digit split, ms[1] = the int8 tcgen05 contraction,
 * ms[2] = the ordered tile reduction.  For benchmarks and profiling.       */
int bmm_segsq_i8_timed(int dtype, const void* A, int64_t lda, int64_t strideA,
                       const void* B, int64_t ldb, int64_t strideB,
                       int64_t m, int64_t nc, int64_t n_inner, const int64_t* seg, int64_t nseg, int64_t seg_stride,
                       int64_t batch, double* gsq, void* ws, int64_t ws_bytes, void* stream, float* ms);

/* C @ D on the int8 tensor cores (the same Ozaki digit planes, one
 * power-of-two scale per row of A / column of B): out[b] = A[b] (m x k) @ B[b]
 * (k x nc) in float64 (estimators.py:175).  k = k_dev[b] <= k_max when k_dev
 * != NULL (the compressed sketch's device count).  kexp (optional, per k,
 * stride k_max per problem): A[:, k] 2^kexp[k], B[k, :] 2^-kexp[k] -- exact
 * balancing that keeps the digit scales set by the dominant terms; without
 * it heavy-tailed operands lose a few bits (~1e-13 relative instead of
 * ~1e-15).  The K dimension is split across CTAs when the output has few
 * tiles; partials are summed in a fixed order (deterministic).  float64 or
 * float32 operands, row-major, lda/ldb in elements.                         */
int64_t bmm_gemm_i8_workspace(int64_t m, int64_t nc, int64_t k_max, int64_t batch);
int bmm_gemm_i8(int dtype, const void* A, int64_t lda, int64_t strideA,
                const void* B, int64_t ldb, int64_t strideB,
                int64_t m, int64_t nc, int64_t k_max, const int64_t* k_dev, const int32_t* kexp, int64_t batch,
                double* out, int64_t ldo, int64_t strideO, void* ws, int64_t ws_bytes, void* stream);
/* The same with the sketch gathered on the fly (estimators.py:78-81):
 * A[h, t] = M[h, column[t]] * scale[t], B[t, f] = N[column[t], f] * scale[t]
 * (one float64 rounding each, as the reference's C and D), column/scale/kexp
 * per problem at b * w_stride.  Workspace: bmm_gemm_i8_workspace(m, nc, k_max, batch). */
int bmm_gemm_i8_gather(int dtype, const void* M, int64_t ldm, int64_t strideM,
                       const void* N, int64_t ldn, int64_t strideN,
                       const int64_t* column, const double* scale, const int32_t* kexp, int64_t w_stride,
                       int64_t m, int64_t nc, int64_t k_max, const int64_t* k_dev, int64_t batch,
                       double* out, int64_t ldo, int64_t strideO, void* ws, int64_t ws_bytes, void* stream);
/* Balance exponents for the above from the norm pass: kexp[b*w_stride + t] =
 * round(log2(||N_i|| / ||M_i||) / 2) with i = column[b*w_stride + t] (t when
 * column is NULL), colsq/rowsq = squared column norms of M / row norms of N
 * (bmm_norms), n_stride per problem; 0 past k_dev[b] and for zero norms.   */
int bmm_balance_exponents(const double* colsq, const double* rowsq, int64_t n_stride,
                          const int64_t* column, int64_t w, int64_t w_stride, const int64_t* k_dev,
                          int64_t batch, int32_t* kexp, void* stream);

/* The same as bmm_segsq_f64_gather through Gram matrices, for segments of few
 * sketch columns (the two-step pilot: c0/K draws per block):
 * ||C_j D_j||_F^2 = sum_{a,a'} (C_j^T C_j)[a,a'] (D_j D_j^T)[a,a'], two streaming
 * passes over the gathered columns instead of an m x p product per segment.
 * plan.py:457-464.  Float64 (float32 inputs upcast), deterministic; parity to
 * rounding like the DMMA kernel.  max_len bounds every segment's length
 * (<= 8: a single-tile variant).  No workspace.                             */
int bmm_segsq_gram_gather(int dtype, const void* M, int64_t ldm, int64_t strideM,
                          const void* N, int64_t ldn, int64_t strideN,
                          int64_t m, int64_t nc, const int64_t* column, const double* scale,
                          int64_t w_stride, const int64_t* seg, int64_t nseg, int64_t seg_stride,
                          int64_t max_len, int64_t batch, double* gsq, void* stream);

/* OPL block-product norms through the Gram identity (K7):
 * gsq[b, j] = || A[:, seg_j] B[seg_j, :] ||_F^2 = < A_j^T A_j , B_j B_j^T >_F,
 * two L x L Gram matrices per segment on the DMMA pipe (36 of the 64 8x8 tiles:
 * symmetry), contraction over the m rows of A and the nc columns of B.
 * Replaces the K dgemm + ddot loop of block_scores (plan.py:176-189) when
 * L < m nc / (m + nc): 2 (m + nc) n L flops instead of 2 m nc n, A and B read
 * once.  Segments up to bmm_segsq_gram_max_len() (64) columns; longer -> NaN.
 * dtype BMM_F64 or BMM_F32 (widened exactly).  No workspace, deterministic
 * (fixed-order warp and lane reductions), result clamped at 0.             */
int64_t bmm_segsq_gram_max_len(void);
int bmm_segsq_gram(int dtype, const void* A, int64_t lda, int64_t strideA,
                   const void* B, int64_t ldb, int64_t strideB,
                   int64_t m, int64_t nc, const int64_t* seg, int64_t nseg, int64_t seg_stride,
                   int64_t batch, double* gsq, void* stream);
/* The same, with the norm pass fused in (round 2): the segments must tile the
 * inner dimension (seg[0] = 0, seg[nseg] = n), and the kernel that reads each
 * segment's columns of A and rows of B once also writes colsq[b*n_stride + i]
 * (column_norms^2, NumPy's sequential order over the m rows, matrix.py:107-109)
 * and rowsq[b*n_stride + i] (row_norms^2, NumPy's pairwise tree over the nc
 * columns, matrix.py:112-114) -- bit-identical to bmm_norms.  nc must be
 * 128 * 2^k (the tree is then perfect: 128-element leaves paired in order).  */
int bmm_segsq_gram_norms(int dtype, const void* A, int64_t lda, int64_t strideA,
                         const void* B, int64_t ldb, int64_t strideB,
                         int64_t m, int64_t nc, const int64_t* seg, int64_t nseg, int64_t seg_stride,
                         int64_t batch, double* gsq, double* colsq, double* rowsq, int64_t n_stride,
                         void* stream);

/* ---------------------------------------------------------------- exact variance analytics
 * (analysis.py:57-116)
 * var[h, f] = sum_i M[h,i]^2 N[i,f]^2 / (c_k p_i)  -  sum_k (M^k N_k)[h,f]^2 / c_k
 * over p_i > 0 and c_k > 0 (elementwise_variance, analysis.py:57-90): one
 * squared-mode DMMA GEMM over the inner dimension, then a segmented GEMM whose
 * epilogue accumulates weighted squares, subtracted in a fixed chunk order.
 * budgets are real-valued (the reference allows a real override).  *bad gets
 * K - k for the first block k with a contributing column of zero probability
 * (analysis.py:77-79 ValueError), 0 if none.  float64 operands.             */
int64_t bmm_variance_workspace(int64_t m, int64_t p, int64_t n, int64_t K);
int bmm_elementwise_variance(const double* M, int64_t ldm, const double* N, int64_t ldn,
                             int64_t m, int64_t n, int64_t p, const int64_t* offsets, int64_t K,
                             const double* probs, const double* colsq, const double* rowsq,
                             const double* budgets, double* var, int64_t ldv, int64_t* bad,
                             void* ws, int64_t ws_bytes, void* stream);
/* out[k] = sum over p_i > 0 in block k of (sqrt(colsq_i) sqrt(rowsq_i))^2 / p_i
 * (expected_sq_error's first term, analysis.py:109); *bad as above
 * (analysis.py:105-107).                                                    */
int bmm_block_term1(const double* probs, const double* colsq, const double* rowsq,
                    const int64_t* offsets, int64_t K, double* out, int64_t* bad, void* stream);

/* ---------------------------------------------------------------- K9 error
 * err[b] = { sum (X - Y)^2, sum X^2 } over m x nc (X = exact MN, Y = C D),
 * float64 accumulation, deterministic two-level reduction.  X, Y may be
 * float64 (dtype F64) or float32 (dtype F32).  analysis.py:318-325.        */
int64_t bmm_sqdiff_workspace(int64_t m, int64_t nc, int64_t batch);
int bmm_sqdiff(int dtype, const void* X, int64_t ldx, int64_t strideX,
               const void* Y, int64_t ldy, int64_t strideY,
               int64_t m, int64_t nc, int64_t batch, double* err,
               void* ws, int64_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- K4/K6 float32 path
 * Split gather: x = M[h, column[t]] * scale[t] (formed in float64, as the
 * reference does on upcast inputs), h = tf32_rna(x), l = x - h:
 *   a_hi[(b*m + h) * W + t]            float32 holding tf32 h   (A = C, K-major)
 *   a_x [(b*m + h) * 2W + 16*(t/8) ..] bf16 pairs [h(8) | l(8)] per 8-column group
 *   b_hi, b_x                          the same for B = D^T, pairs [l(8) | h(8)]
 * W % 8 == 0.  a_x / b_x occupy the same bytes as a float32 W-vector per row. */
int bmm_gather_f32split(int dtype, const void* M, int64_t ldm, int64_t strideM,
                        const void* N, int64_t ldn, int64_t strideN,
                        int64_t m, int64_t p, const int64_t* column, const double* scale,
                        int64_t W, int64_t w_stride, int64_t batch,
                        float* a_hi, void* a_x, float* b_hi, void* b_x, void* stream);

/* out[b] (m x nc, float32) ~= C[b] (m x k) @ D[b] (k x nc) from the split
 * operands: tcgen05.mma kind::tf32 for h_C.h_D plus one kind::f16 (bf16) MMA
 * for both cross terms h_C.l_D + l_C.h_D, float32 TMEM accumulation promoted
 * to round-to-nearest registers every 128 K-elements, TMA SWIZZLE_128B
 * operand tiles (estimators.py:175 for the float32 configs).  k % 8 == 0.   */
int bmm_gemm_f32split(const float* a_hi, const void* a_x, const float* b_hi, const void* b_x,
                      int64_t m, int64_t nc, int64_t k, int64_t batch,
                      float* out, int64_t ldo, int64_t strideO, void* stream);
/* F16 split for the CTA-pair contraction (config 4 sizes): C.D for float32 data
 * (estimators.py:175) with every sketch value x = h + l, h = fp16(y), l = fp16(y - h),
 * y = x * 2^(kexp[t] - gshift[b]) for C and 2^(-kexp[t] - gshift[b]) for D (exact
 * powers of two: the balanced exponents keep both operands inside fp16's range).
 * bmm_balance_f16: kexp from the norm pass (colsq/rowsq, n_stride per problem)
 *   and the sketch scales, gshift per problem so that |y| < 2^15; 0 past k_dev.
 * bmm_gather_f16split_dk: a_h and a_x = the high and the low fp16 halves of C
 *   (rows x W each), b_h / b_x likewise for D^T; columns zero-padded to a multiple
 *   of 64 past k_dev (the contraction's K step).  4 operand bytes per sketch
 *   element; buffers of the float32 split (a_hi/a_x/b_hi/b_x) are large enough.
 * bmm_gemm_f16split_dk: out[b] = 2^(2 gshift[b]) * (a . b^T) on CTA pairs
 *   (tcgen05.mma.cta_group::2, 256 x 256 tiles), per 16 K the three kind::f16
 *   MMAs h.h' + h.l' + l.h'.                                                   */
int bmm_balance_f16(const double* colsq, const double* rowsq, int64_t n_stride, const int64_t* column,
                    const double* scale, int64_t w, int64_t w_stride, const int64_t* k_dev, int64_t batch,
                    int32_t* kexp, int32_t* gshift, void* stream);
int bmm_gather_f16split_dk(int dtype, const void* M, int64_t ldm, int64_t strideM, const void* N,
                           int64_t ldn, int64_t strideN, int64_t m, int64_t p, const int64_t* column,
                           const double* scale, const int32_t* kexp, const int32_t* gshift, int64_t W,
                           int64_t w_stride, const int64_t* w_dev, int64_t batch, void* a_h, void* a_x,
                           void* b_h, void* b_x, void* stream);
int bmm_gemm_f16split_dk(const void* a_h, const void* a_x, const void* b_h, const void* b_x, int64_t m,
                         int64_t nc, int64_t k_max, const int64_t* k_dev, const int32_t* gshift,
                         int64_t batch, float* out, int64_t ldo, int64_t strideO, void* stream);

/* Compressed-sketch variants (bmm_compress_sketch): the gather writes and the
 * contraction reads only the first ceil(count[b] / 32) * 32 sketch columns of
 * problem b (the compression zero-pads the scales past the count).          */
int bmm_gather_f32split_dk(int dtype, const void* M, int64_t ldm, int64_t strideM,
                           const void* N, int64_t ldn, int64_t strideN, int64_t m, int64_t p,
                           const int64_t* column, const double* scale, int64_t W, int64_t w_stride,
                           const int64_t* w_dev, int64_t batch, float* a_hi, void* a_x,
                           float* b_hi, void* b_x, void* stream);
int bmm_gemm_f32split_dk(const float* a_hi, const void* a_x, const float* b_hi, const void* b_x,
                         int64_t m, int64_t nc, int64_t k_max, const int64_t* k_dev, int64_t batch,
                         float* out, int64_t ldo, int64_t strideO, void* stream);
/* The gather and the contraction in ONE kernel (float32 inputs): producer warps
 * gather C = M[:, column] * scale and D = N[column, :] * scale[:, None] (the
 * sketch, estimators.py:78-80 / 244-249), split them (tf32 hi + bf16 pairs, in
 * float32 arithmetic) straight into the swizzled shared-memory stages of the
 * tcgen05 contraction (estimators.py:175), so the split operands never reach
 * HBM.  out[b] = C[b] @ D[b] over the first min(w_dev[b], W) sketch columns
 * (w_dev NULL: all W).  128 x 128 output tiles; dtype BMM_F32 only.          */
int bmm_gemm_f32split_gather(int dtype, const void* M, int64_t ldm, int64_t strideM,
                             const void* N, int64_t ldn, int64_t strideN, int64_t m, int64_t p,
                             const int64_t* column, const double* scale, int64_t W, int64_t w_stride,
                             const int64_t* w_dev, int64_t batch, float* out, int64_t ldo,
                             int64_t strideO, void* stream);

/* The fp16-split form of the same fusion (round 2, config 5): one CTA per
 * 256 x 256 output tile, every element of C and D gathered once per tile,
 * scaled by 2^(kexp[t] - gshift[b]) (C) and 2^(-kexp[t] - gshift[b]) (D) from
 * bmm_balance_f16, split into fp16 h + l and contracted as h.h + h.l + l.h
 * (kind::f16) into an unpromoted TMEM accumulator; out[b] = 2^(2 gshift[b])
 * (C[b] @ D[b]).  The accumulator's truncation error grows with K (~4.5e-9 per
 * sketch column): the pipeline uses it for W <= 1024.  M is streamed by TMA
 * (16-column slabs holding a drawn column): its rows must be 16-byte aligned
 * (ldm, strideM multiples of 4).  dtype BMM_F32 only.                          */
int bmm_gemm_f16split_gather(int dtype, const void* M, int64_t ldm, int64_t strideM,
                             const void* N, int64_t ldn, int64_t strideN, int64_t m, int64_t n, int64_t p,
                             const int64_t* column, const double* scale, const int32_t* kexp,
                             const int32_t* gshift, int64_t W, int64_t w_stride, const int64_t* w_dev,
                             int64_t batch, float* out, int64_t ldo, int64_t strideO, void* stream);

/* ---------------------------------------------------------------- exchanges over NCCL
 * The cross-rank steps of the sharded product (distributed.py; SURVEY §8(b2)
 * optional ncclComm_t variants, §8(e1) C1-C3), enqueued on the caller's stream.
 * NCCL is resolved at run time (libnccl.so.2, the process's own copy when one
 * is loaded); without it these return BMM_E_UNSUPPORTED.  `comm` is an
 * ncclComm_t (opaque here: no NCCL types in the ABI).
 * bmm_nccl_version: NCCL's version code, 0 when unavailable.
 * bmm_nccl_unique_id: ncclGetUniqueId into id_out (128 bytes); rank 0 makes
 *   it, the caller broadcasts it (torch.distributed does it in distributed.py).
 * bmm_nccl_comm_init / _destroy: ncclCommInitRank / ncclCommDestroy.
 * bmm_all_gather_f64_nccl: dst (nranks x len) = every rank's src, rank order
 *   (C1: the colsq chain hand-offs and the rowsq subtree partials).
 * bmm_exchange_sum_nccl: out = ((p_0 + p_1) + p_2) + ... over the ranks'
 *   partials (C2: g_k^2 and pilot^2 over output tiles; C3: error sums) --
 *   an all-gather into ws (nranks x len) and a fixed rank-order sum, so every
 *   rank holds identical bits (replaces distributed.exchange_sum).            */
int bmm_nccl_version(void);
int bmm_nccl_unique_id(void* id_out);
int bmm_nccl_comm_init(void** comm_out, int nranks, const void* id, int rank);
int bmm_nccl_comm_destroy(void* comm);
int bmm_all_gather_f64_nccl(void* comm, const double* src, int64_t len, double* dst, void* stream);
int bmm_exchange_sum_nccl(void* comm, int nranks, const double* partial, int64_t len, double* ws,
                          double* out, void* stream);

/* The whole plan of MANY SMALL problems, one CTA per problem (config 5: 4096 problems of
 * n = 4096, K = 64): bmm_block_probs + bmm_budgets (ONC / OPL rules) + bmm_seed_streams +
 * bmm_sample + bmm_compress_sketch + bmm_balance_f16 in one launch, with the probabilities
 * and the CDF held in shared memory (plan.py:165-206, 242-421; estimators.py:34-44, 78,
 * 141).  Same device functions in the same order as the separate entries: every output is
 * bit-identical to theirs.  cum, last_support, diag, notes, states and (kexp, gshift) are
 * optional (NULL).  Needs blocks of at most 128 columns (max_len: one leaf of NumPy's pairwise
 * sum per block), bmm_plan_small_smem(n, K, W) <= 200 KiB and n, W < 65536; BMM_E_UNSUPPORTED
 * otherwise (callers then use the separate entries).                                        */
int64_t bmm_plan_small_smem(int64_t n, int64_t K, int64_t W);
/* diagnostics: later launches write 16 SM-clock stamps per problem (stage boundaries) to
 * `stamps` (batch x 16, device); NULL switches it off (tools/plan_small_probe.py)          */
int bmm_plan_small_debug(long long* stamps);
int bmm_plan_small(int rule, const double* colsq, const double* rowsq, int64_t n,
                   const int64_t* offsets, const int64_t* sizes, int64_t K, int64_t batch,
                   int64_t max_len, const double* aux, const int64_t* c, int cap, const uint32_t* words,
                   int64_t n_words, const int64_t* first_child, int64_t W, double* probs, double* s,
                   double* cum, int64_t* last_support, int64_t* budgets, int64_t* col_off,
                   int32_t* status, int64_t* diag, int32_t* notes, uint64_t* states,
                   int64_t* column, double* prob, double* scale, int64_t* k_column,
                   double* k_scale, int64_t* k_count, int32_t* kexp, int32_t* gshift, void* stream);

/* Diagnostics: the device clock (%globaltimer, ns) written to out[0] by a
 * one-thread kernel on `stream` (graph-capturable; tools/timeline.py).        */
int bmm_timestamp(unsigned long long* out, void* stream);

/* sum of a float64 vector segment in numpy pairwise order: out[b] = 0 + pw(x[b, 0:len])
 * (used for ||M||_F^2 = pw(colsq), ||N||_F^2 = pw(rowsq)).                */
int bmm_pairwise_sum(const double* x, int64_t len, int64_t stride, int64_t batch,
                     double* out, void* stream);

/* ---------------------------------------------------------------- instances
 * gen_normal_instance / gen_heavy_tail_instance (datagen.py:55-110) on device:
 * M (m x n) columns and N (n x p) rows are AR(1) vectors with covariance
 * scale * rho^|i-j| (datagen.py:38-42), generated by the recursion that equals
 * L @ z for the Cholesky factor L; heavy != 0 divides each vector by
 * sqrt(chi^2(1)) and adds `location`.  Vector j of each side draws from its own
 * PCG64 stream, SeedSequence-hashed from (seed_lo, seed_hi, side tag) with child
 * j; normals by Box-Muller.  Deterministic per seed; distribution-identical to,
 * not bit-identical with, the reference's numpy draws.  Either output may be
 * NULL.  dtype BMM_F64 or BMM_F32 (generated in float64, rounded once).      */
int bmm_gen_instance(int heavy, int dtype, int64_t m, int64_t n, int64_t p,
                     uint64_t seed_hi, uint64_t seed_lo,
                     double scale_left, double rho_left, double scale_right, double rho_right,
                     double location, void* M, int64_t ldm, void* N, int64_t ldn, void* stream);

/* The same instances from the REFERENCE's own variates (datagen.py:70-71, 104-106):
 * Z (dim x count, row-major float64, device) holds rng.standard_normal((dim, count)) as the
 * reference draws it -- numpy's ziggurat/gamma variates are third-party libm-dependent
 * arithmetic, so the caller's Generator produces them and the generator state advances
 * exactly as in the reference -- and this entry replaces the Cholesky product L @ Z by the
 * AR(1) recursion: out[i, j] (transpose_out = 0: M, dim = m, count = n) or out[j, i]
 * (transpose_out = 1: N = ascontiguousarray((L @ Z).T), dim = p, count = n).  w_opt (count
 * chi-square(1) draws, device) selects the heavy-tailed form location + x / sqrt(w[j]) in the
 * reference's operation order.  dtype of out: BMM_F64 or BMM_F32 (rounded once).           */
int bmm_ar1_transform(int dtype, const double* Z, int64_t dim, int64_t count, int64_t ldz,
                      int transpose_out, double scale, double rho, const double* w_opt,
                      double location, void* out, int64_t ldo, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BLOCKMM_B200_H */
