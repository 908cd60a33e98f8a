/*
 * bs.h: C ABI of the B200 balanced-sparsity library (libbs.so).
 *
 * The library implements the inference hot path of "Balanced Sparsity for Efficient DNN Inference
 * on GPU" (arXiv 1811.00206; /root/reference/PAPER.md, cited as P:<line>). That path is the product
 * of a balanced-sparse weight matrix and dense activations:
 *   - the FC layer Y = W·X + B of Eq. 1, with bias B = 0 as in the analysis;
 *   - W pruned to Balanced Sparsity: "each matrix row is split into multiple equal-sized blocks and
 *     each block has the same number of non-zero weights";
 *   - one block partition's multiply-accumulates go to one thread;
 *   - x is rearranged in shared memory so that the gathers hit distinct banks.
 *
 * Conventions (every entry point):
 *   - Device pointers are caller-owned (allocated by PyTorch or cudaMalloc). The library never
 *     allocates device memory and keeps no state beyond a per-device property cache.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream). Every device call
 *     is asynchronous and stream-ordered; none synchronises.
 *   - Arguments are validated synchronously, before anything is enqueued. A failed check returns a
 *     status != BS_OK and enqueues nothing. Launch failures return BS_ERR_CUDA. Asynchronous device
 *     faults surface at the caller's next synchronisation, as usual in CUDA.
 *   - Inputs must not alias outputs.
 *   - Results are deterministic: the same inputs give bit-identical outputs. No reduction uses atomics.
 *   - Storage layouts (canonical, SPMV, SPMM, SP24) are specified in docs/layout.md.
 *   - Value, x and y dtypes are equal. Accumulation is fp32.
 */
#ifndef BS_H_
#define BS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BS_OK = 0,
  BS_ERR_ARG = 1,         /* null pointer, k outside [0,B], sparsity outside [0,1), N < 1, bad ld */
  BS_ERR_SHAPE = 2,       /* K mod B != 0 ("equal-sized blocks"; rejected, not padded), M/K < 1 */
  BS_ERR_DTYPE = 3,       /* unknown dtype code */
  BS_ERR_UNSUPPORTED = 4, /* valid but not implemented: B > 65536, SP24 with B != 4 or k != 2, ... */
  BS_ERR_CUDA = 5         /* a CUDA runtime call or kernel launch failed */
} bs_status;

typedef enum { BS_F32 = 0, BS_F16 = 1, BS_BF16 = 2 } bs_dtype;

typedef enum { BS_LAYOUT_SPMV = 1, BS_LAYOUT_SPMM = 2, BS_LAYOUT_SP24 = 3 } bs_layout;

/* A packed balanced-sparse matrix: M×K, blocks of width `block`, `k` kept per block, values of
 * dtype `dt`, stored in `layout` at device pointer `packed` (bs_packed_bytes bytes). */
typedef struct {
  int64_t M, K;
  int32_t block, k;
  int32_t dt;      /* bs_dtype */
  int32_t layout;  /* bs_layout */
  const void* packed;
} bs_matrix;

/* ---------------------------------------------------------------- host helpers (pure, sync) */

/* Kept entries per block for a nominal sparsity s: k = lround((1 - s) * block), computed in IEEE
 * double with round-half-away-from-zero. Alg. 1 zeros "a fraction of weights with smallest absolute
 * magnitudes", and every block keeps the same count. The rounding rule is
 * SURVEY reading A1, pinned by P:95 (4, 0.5 -> 2), P:409 (32, 0.9 -> 3) and P:380 (32, 0.875 -> 4).
 * Returns -1 if block < 1 or s is outside [0, 1). */
int bs_k_from_sparsity(int block, double sparsity);

/* Bytes of a packed buffer in `layout` (docs/layout.md). Returns 0 on invalid arguments. */
size_t bs_packed_bytes(int64_t M, int64_t K, int block, int k, int dt, int layout);

/* The layout bs_spmm runs fastest on for a batch of N columns, from the round-1 measurements
 * (bench.py `spmm`): the 2:4 shape (block 4, k 2, f16/bf16, K mod 128 = 0) -> SP24
 * (sparse tensor cores for N >= 2, a CUDA-core SpMV at N = 1); otherwise N <= 8, or N <= 16 with
 * K <= 3072, -> SPMV (the batched CUDA-core path streams W once per 8 or 16 columns) and larger
 * batches with f16/bf16 and block | 64 -> SPMM
 * (decompressed tiles on tcgen05.mma); f32 -> SPMV. The choice depends only on the arguments, never on
 * the data, and every layout gives results within the same tolerance. Returns -1 on invalid arguments. */
int bs_choose_layout(int64_t M, int64_t K, int block, int k, int dt, int64_t N);

/* Introspection for the bank-conflict model (tests/test_bank_model.py): the byte offset, within the
 * shared-memory x slots of bs_spmv (nv = 1) or of a bs_spmm pass of nv columns on the SPMV layout
 * (nv = 2, 4, 8, 16; 16-bit dtypes), of the `part`-th shared-memory load that gathers element
 * (block b, offset o) of x (part 0, or 0 and 1 for nv = 16: two 16-byte loads). This is the paper's
 * rearranged x (Fig. 3): the kernel stages and gathers x through the same functions.
 * Returns -1 on invalid arguments. Host, pure. */
int64_t bs_x_slot_offset(int64_t K, int block, int dt, int nv, int64_t b, int o, int part);

/* Human-readable status name. */
const char* bs_status_str(int status);

/* Library build string: compile target and version. */
const char* bs_version(void);

/* ---------------------------------------------------------------- device work (async) */

/* bs_prune_k: one balance-aware pruning step (Alg. 1 inner loop, with the count-based
 * reading A2 that guarantees P:94's "same number of non-zero weights"). For every row r and block b
 * it keeps the k entries of W[r][b·B .. b·B+B) with the largest magnitude (ties -> lower offset,
 * NaN above Inf; docs/layout.md "Canonical form").
 *   W     device, M×K of dtype dt, row-major, leading dimension ldw >= K elements
 *   vals  device out, [M][K/B][k] of dt: bit copies of the kept weights
 *   idx   device out, [M][K/B][k] of uint16: kept block-local offsets, ascending
 * Errors: BS_ERR_SHAPE if K mod B != 0; BS_ERR_ARG if k not in [0,B] or ldw < K or a pointer is NULL
 * (vals/idx may be NULL only when k == 0); BS_ERR_UNSUPPORTED if B > 65536. */
int bs_prune_k(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int block, int k,
               void* vals, uint16_t* idx, void* stream);

/* bs_prune: bs_prune_k with k = bs_k_from_sparsity(block, sparsity). The k used is written to
 * *k_out (a host int; may be NULL). BS_ERR_ARG if sparsity is outside [0,1). */
int bs_prune(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int block, double sparsity,
             int* k_out, void* vals, uint16_t* idx, void* stream);

/* bs_block_rank: every element's position in its block's magnitude order (Alg. 1 "sorts the weights in
 * each block by their absolute magnitude"; ties to the lower offset, NaN above Inf, as
 * bs_prune_k). A pruning step at any k keeps exactly the entries with rank < k, so one pass yields the
 * masks of a whole gradual sparsity schedule (Alg. 1's outer loop) without retraining.
 *   W     device, M×K of dtype dt, row-major, leading dimension ldw >= K elements
 *   rank  device out, M×K uint8 (row-major, leading dimension K); any alignment (32-bit stores are
 *         used only when rank is 4-byte aligned)
 * Errors: as bs_prune_k; BS_ERR_UNSUPPORTED unless block is 1, 2, 4, 8, 16 or 32. */
int bs_block_rank(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int block, uint8_t* rank,
                  void* stream);

/* ---------------------------------------------------------------- Alg. 1's schedule and the comparison patterns */

/* GraduallyIncrease (Alg. 1): the threshold sparsity of pruning iteration i of n. The paper says
 * only that it "is gradually increased from 0 to the target sparsity while the increase rate decreases
 * with pruning iteration"; the trajectory is SPEC's cubic (reading A20):
 *   s_i = target · (1 - (1 - i/n)^3),  i = 0..n   (s_0 = 0, s_n = target: 0.9, 10, 5 -> 0.7875).
 * Host, pure. Returns -1 if n < 1, i outside [0, n] or target outside [0, 1). */
double bs_schedule_sparsity(double target, int n, int i);

/* Units kept at sparsity s by the global patterns below: lround((1 - s) · n), the rounding of k
 * (reading A1 applied to the whole unit count, A8, A22). Host, pure. -1 on bad arguments. */
int64_t bs_keep_count(int64_t n, double sparsity);

/* bs_decode: the dense W_bs, i.e. Alg. 1's output "the pruned matrix M_p", from canonical
 * (vals, idx): W[r][b·B + idx[r][b][t]] = vals[r][b][t] (bit copies), +0 everywhere else.
 * bs_prune_k followed by bs_decode is one pruning iteration of Alg. 1 on a dense matrix (in place
 * when W is the pruned matrix itself: bs_prune_k reads it completely before bs_decode writes, in
 * stream order); iterating it along bs_schedule_sparsity is Alg. 1's schedule without retraining.
 *   vals, idx  device, canonical [M][K/B][k] (bs_prune_k's output)
 *   W          device out, M×K of dtype dt, row-major, leading dimension ldw >= K
 * Errors: as bs_pack for the shape arguments; BS_ERR_ARG for NULL pointers or ldw < K. */
int bs_decode(const void* vals, const uint16_t* idx, int64_t M, int64_t K, int block, int k, int dt,
              void* W, int64_t ldw, void* stream);

/* Device scratch the mask generators below need (bh = bw = 0 for bs_random_mask): selection state,
 * per-CTA counters and, for tiles, one 8-byte score and one byte per tile. Host, pure. */
size_t bs_pattern_workspace_bytes(int64_t M, int64_t K, int64_t bh, int64_t bw);

/* bs_random_mask: random sparsity, the paper's main comparison pattern (Han et al.; P:39, P:230,
 * "performs pruning in each independent weight matrix"): magnitude pruning over the WHOLE
 * matrix, mask[r·K + c] = 1 for the bs_keep_count(M·K, s) entries of largest |w| (the magnitude key of
 * bs_prune_k: NaN above Inf; ties -> lower row-major index), 0 elsewhere.
 *   W          device, M×K of dt, leading dimension ldw >= K;  mask  device out, M×K uint8
 *   workspace  device scratch of at least bs_pattern_workspace_bytes(M, K, 0, 0) bytes
 * A radix select over the keys (integer decisions only: the mask is exact).
 * Errors: BS_ERR_ARG for bad sparsity, NULL pointers, ldw < K or a short workspace. */
int bs_random_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, double sparsity, uint8_t* mask,
                   void* workspace, size_t workspace_bytes, void* stream);

/* bs_block_mask: block sparsity (Narang et al., Table brange's 4×4 / 8×8 / 16×16):
 * bh×bw tiles in row-major tile order, each scored by "the maximum magnitude or the average magnitude
 * of the weights within one block as a representative":
 *   criterion 0: max |w| (as the magnitude key: NaN above Inf);
 *   criterion 1: mean |w|, compared as the fp64 sum of |w| taken in row-major order inside the tile
 *                (the mean times the fixed tile size; any NaN ranks the tile above all others).
 * The bs_keep_count(#tiles, s) best tiles are kept whole (ties -> lower tile index); mask as above.
 * Vector sparsity (Mao et al.; "a whole row or column ... as a basic pruning unit") is this call
 * with bh = 1, bw = K (rows) or bh = M, bw = 1 (columns) and criterion 1.
 * Errors: BS_ERR_SHAPE if M mod bh or K mod bw != 0; BS_ERR_ARG as bs_random_mask or criterion not 0/1. */
int bs_block_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int64_t bh, int64_t bw,
                  double sparsity, int criterion, uint8_t* mask, void* workspace, size_t workspace_bytes,
                  void* stream);

/* bs_im2col: convolution as matrix multiplication, "using im2col that converts convolution operation to
 * matrix-matrix multiplication", so that a conv layer whose kernels form one balanced-sparse
 * weight matrix runs as bs_spmm (NEXT-3: N = pixels, the large-N regime of the tensor-core paths).
 * Activations are NHWC (channels last); the weight matrix is Cout × (kh·kw·C) with columns in (dy, dx, c)
 * order (torch weight.permute(0, 2, 3, 1); reading A23). Then bs_spmm(A, X) = Y [pixels][Cout]
 * is the NHWC output.
 *   in  device, [Nimg][H][W][C] of dt;  X  device out, [Nimg·OH·OW] rows of kh·kw·C elements, row stride ldx
 *   X[(n·OH + oy)·OW + ox][(dy·kw + dx)·C + c] = in[n][oy·stride + dy - pad][ox·stride + dx - pad][c],
 *   +0 outside the image; OH = (H + 2·pad - kh)/stride + 1, OW likewise. A pure copy (bit-exact).
 * Errors: BS_ERR_SHAPE for non-positive sizes or a kernel larger than the padded image; BS_ERR_ARG for
 * NULL pointers or ldx < kh·kw·C. */
int bs_im2col(const void* in, int dt, int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh, int kw, int pad,
              int stride, void* X, int64_t ldx, void* stream);

/* bs_spmm_fused: a fully connected layer at batch N, Y = act(W_bs·X + bias) (Eq. 1 with its +B; the VGG
 * classifier layers at batch), on the tensor cores: layout SPMM (block | 64) or SP24 (K % 128 ==
 * 0), f16/bf16, X rows 16-byte aligned with ldx % 8 == 0. bias: M elements of A's dtype or NULL; act: bs_act, applied in fp32
 * before the one rounding (bs_spmv_fused's expressions). With bias = NULL and act = BS_ACT_NONE the result
 * is bit-identical to bs_spmm on the same operands. X, Y as bs_spmm.
 * Errors: as bs_spmm; BS_ERR_ARG for an unknown act; BS_ERR_UNSUPPORTED when the operands are not eligible. */
int bs_spmm_fused(const bs_matrix* A, const void* X, int64_t N, int64_t ldx, const void* bias, int act, void* Y,
                  int64_t ldy, void* stream);

/* bs_conv2d: a convolution layer as one balanced-sparse product with implicit im2col ("im2col that
 * converts convolution operation to matrix-matrix multiplication"; all kernels of a layer form one
 * weight matrix): Y [Nimg·OH·OW][M] = W_bs · im2col(in)ᵀ, i.e. the NHWC output [Nimg][OH][OW][Cout = M],
 * with in NHWC [Nimg][H][W][C] (16-bit, 16-byte aligned) and W_bs's columns in (dy, dx, c) order (reading
 * A23; A->K = kh·kw·C). The tensor cores' X tiles are loaded straight from `in` by TMA in im2col mode, so
 * no [pixels][kh·kw·C] intermediate exists; the result is bit-identical to bs_im2col + bs_spmm.
 * Requirements: layout SPMM (block | 64; K6) or SP24 (kh·kw·C % 128 == 0; K5, the 2:4 sparse tensor cores),
 * f16/bf16, C % 64 == 0, stride 1. Y has room for
 * Nimg·OH·OW·M elements of A's dtype (caller-owned).
 * Layer epilogue (Eq. 1's +B, and the activation that follows a VGG conv layer): `bias` (M elements
 * of A's dtype, one per output channel, or NULL) is added and `act` (bs_act) applied in fp32 before the
 * one rounding to A's dtype, with bs_spmv_fused's expressions. bias = NULL and act = BS_ACT_NONE give the
 * plain product.
 * Errors: BS_ERR_SHAPE for inconsistent shapes; BS_ERR_ARG for NULL pointers or an unknown act;
 * BS_ERR_UNSUPPORTED when an eligibility condition fails (use bs_im2col + bs_spmm then); BS_ERR_CUDA on a
 * launch failure. */
int bs_conv2d(const bs_matrix* A, const void* in, int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh, int kw,
              int pad, int stride, const void* bias, int act, void* Y, void* stream);

/* bs_pack: permute canonical (vals, idx) into the device layout `layout` and narrow the indices
 * (docs/layout.md: u8 for block <= 256, u16 above; in SPMV panels of 16-bit values with V = 8, 5-bit index
 * runs for block == 32 and 4-bit runs for block <= 16). This is a pure permutation, so the output is
 * byte-exact. The paper stores "the
 * same number of non-zero values in each block partition", so the format needs no row
 * pointers. `packed` receives bs_packed_bytes(...) bytes; alignment padding bytes are zeroed.
 * Errors: as bs_prune_k; BS_ERR_UNSUPPORTED for SP24 unless block == 4, k == 2 and K mod 8 == 0. */
int bs_pack(const void* vals, const uint16_t* idx, int64_t M, int64_t K, int block, int k, int dt,
            int layout, void* packed, void* stream);

/* bs_unpack: the inverse of bs_pack (used by tests: unpack(pack(c)) == c). */
int bs_unpack(const void* packed, int64_t M, int64_t K, int block, int k, int dt, int layout,
              void* vals, uint16_t* idx, void* stream);

/* bs_spmv: y = W_bs · x (Eq. 1, with B = 0; batch 1). A must be in layout SPMV
 * (BS_ERR_UNSUPPORTED otherwise).
 *   x  device, K elements of A->dt;  y  device out, M elements of A->dt.
 * Products are exact in fp32 for f16/bf16, and accumulation is fp32 in a fixed order that does not
 * depend on the row range (so row-sharded results are bit-identical). y is rounded to nearest even.
 * Errors: BS_ERR_ARG for NULL pointers or a bad descriptor; BS_ERR_UNSUPPORTED for an unsupported
 * layout. */
int bs_spmv(const bs_matrix* A, const void* x, void* y, void* stream);

/* Launch flags of bs_spmv_ex.
 * BS_SPMV_PDL: launch as a programmatic dependent of the kernel before it on `stream` (PDL). The
 *   kernel's prologue (shared-memory set-up) overlaps the previous kernel's tail; every global read
 *   and write still waits for the previous kernel to complete (griddepcontrol.wait), so the call is
 *   stream-ordered exactly like a plain launch. bs_spmv uses this flag.
 * BS_SPMV_W_STATIC (with BS_SPMV_PDL): the caller promises that no kernel still running on `stream`
 *   writes A->packed (weights are static, the inference case). The packed W then starts streaming
 *   into shared memory before the wait; x and y still wait. The paper's batch-1 time is dominated by
 *   fixed per-layer costs ("communication inside GPU"; o_time), which this hides. */
/* BS_SPMV_RING: always use the streaming-ring kernel. By default rows of at most 2 KB of packed bytes
 *   (the latency-regime layers) take a direct warp-per-row kernel; the two kernels sum in the same
 *   order, so results are bit-identical either way (this flag exists for tests and A/B timing). */
#define BS_SPMV_PDL 1u
#define BS_SPMV_W_STATIC 2u
#define BS_SPMV_RING 4u

/* bs_spmv_ex: bs_spmv with launch flags (above). flags = BS_SPMV_PDL is bs_spmv; flags = 0 is a
 * plain launch. Errors: as bs_spmv; BS_ERR_ARG for unknown flag bits. Results are bit-identical for
 * every flag combination. */
int bs_spmv_ex(const bs_matrix* A, const void* x, void* y, unsigned flags, void* stream);

/* Activations of the fused layer epilogue. */
typedef enum { BS_ACT_NONE = 0, BS_ACT_RELU = 1, BS_ACT_SIGMOID = 2, BS_ACT_TANH = 3 } bs_act;

/* bs_spmv_fused: the whole layer of Eq. 1, Y = W·X + B, at batch 1 with an activation:
 *   y[r] = act( (W_bs · x)[r] + bias[r] )
 * computed in fp32 (the product exactly as bs_spmv, then + bias, then act: max(v, 0), 1/(1+e^-v) or
 * tanh v) and rounded once to A->dt. The epilogue is fused into the SpMV kernel: the CTA's bias rows
 * are staged in shared memory beside x, so no extra kernel or HBM pass runs.
 *   bias  device, M elements of A->dt, or NULL (no bias);  act  a bs_act value;  flags  as bs_spmv_ex.
 * With bias = NULL and act = BS_ACT_NONE the result is bit-identical to bs_spmv_ex.
 * Errors: as bs_spmv_ex; BS_ERR_ARG for an unknown act; BS_ERR_UNSUPPORTED for layout SP24. */
int bs_spmv_fused(const bs_matrix* A, const void* x, const void* bias, int act, void* y, unsigned flags,
                  void* stream);

/* bs_lstm_step: one step of an LSTM layer whose gate weights are balanced-sparse, in ONE kernel: the
 * gate rows' SpMV with the cell applied in its epilogue. The recurrent workloads of the paper are LSTMs
 * (PTB "2-layer LSTM ... 1500 hidden units", P:347 = BJ.configs[1]'s 6000 x 3000 [W_ih | W_hh];
 * TIMIT Bi-LSTM, hidden 1024). The gate pre-activations are Eq. 1 with its +B:
 *   z = W_bs · x + pre + bias
 * with A's rows interleaved by unit: row 4j + g is gate g (0 input, 1 forget, 2 cell, 3 output) of
 * hidden unit j (a row permutation applied before pruning, which is per row, so it commutes with it).
 * Then, in fp32: i, f, o = sigmoid(z), g = tanh(z_g);  c_out[j] = f·c_prev[j] + i·g;
 * h_out[j] = o·tanh(c_out[j]), rounded once to A->dt.
 *   x       device, K elements of A->dt: [x_t ; h_{t-1}] for A = [W_ih | W_hh], or h_{t-1} for A = W_hh
 *           with pre = W_ih·x_t computed ahead for all steps at once (one bs_spmm with N = T)
 *   pre     device, M elements of A->dt, or NULL;  bias  device, M elements of A->dt, or NULL
 *   c_prev  device, M/4 fp32;  c_out  device out, M/4 fp32;  h_out  device out, M/4 of A->dt
 *   flags   as bs_spmv_ex. No output may alias an input (h_out must not point into x: use two
 *           buffers and alternate them between steps).
 * Errors: as bs_spmv_ex; BS_ERR_SHAPE if M mod 4 != 0; BS_ERR_UNSUPPORTED unless layout SPMV. */
int bs_lstm_step(const bs_matrix* A, const void* x, const void* pre, const void* bias, const float* c_prev,
                 void* h_out, float* c_out, unsigned flags, void* stream);

/* ---------------------------------------------------------------- multi-GPU: the all-gather fused into the SpMV */

/* A row-sharded layer: rank r owns the rows [row0, row0 + A->M) of the M_total-row W_bs and
 * every rank needs the whole y. bs_spmv_allgather computes the shard's rows and, in the same kernel,
 * stores them straight into every rank's full y through peer-mapped pointers (NVLink / NVSwitch P2P);
 * no separate collective runs (NEXT-1). Protocol per call (epoch e = 1, 2, ...):
 *   1. each CTA parks its rows in shared memory, stores its contiguous run into y[p] + row0 for every
 *      rank p, fences at system scope and increments *counter (this rank's, monotonic);
 *   2. the CTA that brings *counter to e·(its grid size) fences again and stores e (release, system
 *      scope) into flags[p][rank] on every rank p;
 *   3. bs_allgather_wait (on each rank's stream) spins, acquire, until flags[rank][q] >= e for all q;
 *      then the whole y of epoch e is visible to the kernels that follow on that stream.
 * Buffers: y[p] (M_total elements of the dtype) and flags[p] (nranks uint32, zeroed before epoch 1) live
 * on rank p and are mapped into every rank (bs_peer_export / bs_peer_import); counter is nranks-local
 * (one uint32, zeroed before epoch 1). A rank must have consumed y of epoch e before it issues the
 * SpMV of epoch e + 2 into the same buffer; alternating two y buffers by epoch parity makes that hold
 * whenever each rank's stream orders its consumption of y_e before its epoch e + 1 wait (the Python
 * FusedRowShardedBS does this). Epochs run to 2^32 / grid (about 29 million calls at 148 CTAs). */
typedef struct {
  int32_t nranks;     /* 1..8 */
  int32_t rank;
  int64_t row0;       /* global row of this shard's first row */
  void* y[8];         /* every rank's full y, mapped into this process */
  uint32_t* flags[8]; /* every rank's arrival flags (nranks words), mapped into this process */
  uint32_t* counter;  /* this rank's CTA completion counter */
  uint32_t epoch;     /* >= 1, incremented by one per call */
} bs_allgather;

/* y (every rank's, rows row0..row0 + A->M) = A·x, with bias/act as bs_spmv_fused (bias of A->M rows, or
 * NULL; act a bs_act). Layout SPMV. Errors: as bs_spmv_fused; BS_ERR_ARG for a bad bs_allgather. */
int bs_spmv_allgather(const bs_matrix* A, const void* x, const void* bias, int act, const bs_allgather* ag,
                      unsigned flags, void* stream);

/* Enqueues the wait of step 3 on `stream` (one tiny kernel). */
int bs_allgather_wait(const bs_allgather* ag, void* stream);

/* Peer mapping of a device buffer between processes of one node (CUDA IPC; the plumbing of
 * bs_allgather). export: a 64-byte handle for the allocation that holds ptr, and ptr's byte offset in it.
 * import: maps a handle exported by another process and returns the pointer at `offset` in it.
 * close: unmaps an imported pointer. No device memory is allocated. */
int bs_peer_export(const void* ptr, void* handle, int64_t* offset);
int bs_peer_import(const void* handle, int64_t offset, void** ptr);
int bs_peer_close(void* ptr, int64_t offset);

/* bs_spmv_host: the same product with HOST x and y. The call enqueues H2D(x) -> bs_spmv -> D2H(y) on
 * `stream`, using caller-owned device scratch x_dev (K elements) and y_dev (M elements). x_host and
 * y_host should be pinned for the copies to be asynchronous. The call does not synchronise: y_host
 * is valid after the stream is synchronised. */
int bs_spmv_host(const bs_matrix* A, const void* x_host, void* y_host, void* x_dev, void* y_dev,
                 void* stream);

/* bs_spmm: Y = W_bs · X for a batch of N columns (Fig. `benchmark`(b), "batchsize = 8").
 *   X  device, column n at X + n·ldx (K elements each), i.e. torch [N, K] with row stride ldx
 *   Y  device out, column n at Y + n·ldy (M elements each), i.e. torch [N, M]
 * Layout SPMM (128-row tiles): f16/bf16 with B dividing 64 run on the tensor cores (tcgen05.mma,
 * decompressed W tiles, fp32 accumulate in tensor memory); other cases use CUDA cores. Layout SPMV:
 * passes of up to 16 columns through the SpMV kernel (16-bit), one SpMV per column (f32). Layout
 * SP24: the sparse tensor cores (tcgen05.mma.sp) at every N, including N = 1 (bs_spmv is the batch-1
 * CUDA-core path; its order differs).
 * Column n of Y depends only on column n of X, with a fixed order of fp32 accumulation over K that
 * does not depend on N, so batch-sharded SpMM reproduces the unsharded columns bit for bit. The order
 * does depend on the operand class: the tensor-core layouts need X rows 16-byte aligned with
 * ldx % 8 == 0 (contiguous torch tensors with K % 8 == 0) and otherwise take a CUDA-core kernel;
 * shards compared bit for bit must share that class.
 * Errors: BS_ERR_ARG if N < 1, ldx < K or ldy < M. */
int bs_spmm(const bs_matrix* A, const void* X, int64_t N, int64_t ldx, void* Y, int64_t ldy,
            void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BS_H_ */
