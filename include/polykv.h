/*
 * polykv.h — C ABI of libpolykv.so, the B200 (sm_100a) SharedKVPool codec.
 *
 * This is the drop-in boundary for PolyKV's compress/inject hot path. The
 * reference (kvpool, pure Python/numpy) has no native interface; each entry
 * point below replaces the numpy function cited next to it, and the Python
 * package `paper_2604_24971_b200` binds them with ctypes so that the
 * reference's public API (kvpool.__all__, /root/reference/pkg/src/kvpool/
 * __init__.py:73-132) keeps its names, arguments and exceptions.
 *
 * Conventions
 *  - Every pointer to tensor data is a DEVICE pointer unless the parameter
 *    name ends in `_host`. Arrays of per-layer pointers (`const void* const*`)
 *    are HOST arrays of device pointers, one entry per layer; they are copied
 *    by value into the kernel parameter block, so they may be freed as soon
 *    as the call returns.
 *  - The library never allocates or frees device memory and keeps no global
 *    mutable state: every entry is reentrant and only enqueues work on the
 *    caller's `stream` (a cudaStream_t passed as void*; NULL = legacy stream).
 *  - Return value: PKV_OK (0) or a negative PKV_ERR_* code. Data faults found
 *    on the device (non-finite input, fp16 scale overflow) are reported as
 *    PKV_FLAG_* bits OR-ed into a caller-provided device status word per
 *    layer, so the caller can check a whole build with a single sync.
 *  - Tensor layout is the reference's: [batch, kv_heads, seq_len, head_dim]
 *    row-major per layer (kvpool/model.py:78-80). `num_vectors` is
 *    batch*kv_heads*seq_len.
 */
#ifndef POLYKV_H_
#define POLYKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PKV_ABI_VERSION 4

/* status codes */
#define PKV_OK 0
#define PKV_ERR_INVALID_ARG (-1)
#define PKV_ERR_UNSUPPORTED_HEAD_DIM (-2)
#define PKV_ERR_CUDA (-3)
#define PKV_ERR_WORKSPACE (-4)
#define PKV_ERR_ALIGNMENT (-5)
#define PKV_ERR_UNSUPPORTED_CODEBOOK (-6)

/* element types */
#define PKV_F32 0
#define PKV_BF16 1

/* key scale modes */
#define PKV_K_TENSOR 0  /* one f32 scale per layer tensor (kvpool/keyquant.py:52-65) */
#define PKV_K_BLOCK32 1 /* one fp16 scale per 32 contiguous elements (q8_0) */

/* device status bits (per layer) */
#define PKV_FLAG_K_NONFINITE 0x1u
#define PKV_FLAG_V_NONFINITE 0x2u
#define PKV_FLAG_K_SCALE_OVERFLOW 0x4u
#define PKV_FLAG_BAD_CODE 0x8u /* pkv_pack_codes: a code > 7 (CorruptBlockError) */

/* Maximum layers handled by one kernel launch; larger pools are processed
 * in consecutive launches by the same call. */
#define PKV_MAX_LAYERS_PER_LAUNCH 64

int pkv_abi_version(void);
const char* pkv_status_string(int status);

/* Scheduling knobs (PKV_KEY_SM_FRACTION, PKV_DEC_KEY_FRACTION, PKV_KEY_LAG,
 * PKV_ATTN_CTAS_PER_SM, PKV_CODEC_PATH, PKV_DBG_ENC) are
 * read from the environment once, at the first launch, not per call. This
 * re-reads them (for A/B tuning in one process). None changes a result. */
int pkv_reload_tuning(void);

/* The last failing CUDA runtime / driver call of the CALLING HOST THREAD,
 * as "<call>: <error name> (<error string>)", or "" if none failed. Set
 * whenever an entry point returns PKV_ERR_CUDA; not cleared by later
 * successful calls. (No reference counterpart: the reference is CPU numpy.) */
const char* pkv_last_cuda_error(void);

/* Head dims supported by the value kernels: 1, 2, 4 (thread-per-word exact
 * kernels), 8 .. 256 (tiled kernels; 64 and 128 streamed through TMA).
 * Key kernels accept any head_dim. Returns 1 if supported. */
int pkv_v_head_dim_supported(int head_dim);

/* Bytes of device workspace pkv_encode needs for `num_layers` layers of
 * `num_vectors` head vectors of `head_dim` (per-layer key maxima are staged
 * there, one 64-bit word per 16384 key elements). */
size_t pkv_encode_workspace_bytes(int num_layers, int64_t num_vectors, int head_dim);

/*
 * pkv_encode — write side of the pool for `num_layers` layers in one launch.
 * Replaces, per layer, kvpool.keyquant.quantize_k (keyquant.py:52-65) and
 * kvpool.valuequant.quantize_v (valuequant.py:193-219) followed by
 * pack_indices_3bit (valuequant.py:312-328), i.e. the loop body of
 * kvpool.pool.build_pool (pool.py:271-273).
 *
 *  k_in / v_in       per-layer input tensors (f32 or bf16, `in_dtype`); either
 *                    array may be NULL to skip that half.
 *  k_mode            PKV_K_TENSOR: k_scale[l] -> 1 float;
 *                    PKV_K_BLOCK32: k_bscale[l] -> ceil(n/32) fp16 bits.
 *  k_codes[l]        int8 codes, one per element.
 *  v_packed[l]       3-bit codes, 8 per 3 bytes, little-endian bit order, over
 *                    the flattened tensor (the PKVP packed payload).
 *  v_scales[l]       f32 RMS per head vector.
 *  centroids_host    8 strictly increasing f32-representable centroids (f64).
 *  sign_bits_host    NULL, or head_dim bits (LSB-first uint32 words): bit i set
 *                    = coordinate i multiplied by -1 before the rotation
 *                    (kvpool.valuequant.sign_diagonal, valuequant.py:183-190).
 *  status            device uint32[num_layers], OR-ed with PKV_FLAG_* bits.
 *  replay_count      device uint32[1] or NULL: incremented once per head vector
 *                    that was re-coded on the exact fp64 path.
 *  k_layer_max       NULL (the per-tensor key scale comes from this call's
 *                    own max|K| pass), or device uint32[num_layers]: the f32
 *                    bit patterns of max|K| per layer computed elsewhere --
 *                    e.g. MAX-reduced over the GPUs that each hold some of a
 *                    layer's KV heads (pkv_k_absmax + an all-reduce); the
 *                    scale is then f32(max/127) exactly as keyquant.py:55-60.
 *                    Ignored for PKV_K_BLOCK32.
 *  workspace         device scratch of pkv_encode_workspace_bytes(num_layers,
 *                    num_vectors, head_dim).
 */
int pkv_encode(int num_layers, int64_t num_vectors, int head_dim, int in_dtype,
               const void* const* k_in, const void* const* v_in, int k_mode,
               int8_t* const* k_codes, float* const* k_scale,
               uint16_t* const* k_bscale, uint8_t* const* v_packed,
               float* const* v_scales, const double* centroids_host,
               const uint32_t* sign_bits_host, uint32_t* status,
               uint32_t* replay_count, const uint32_t* k_layer_max,
               void* workspace, size_t workspace_bytes, void* stream);

/*
 * pkv_k_absmax — max|K| of each of `num_layers` key tensors of `count`
 * elements (f32 or bf16), as f32 bit patterns in device uint32 max_bits[l]
 * (zeroed first; NaN inputs give a pattern above +inf). The per-rank half of
 * keyquant.py:55 when a layer's heads are sharded over GPUs.
 */
int pkv_k_absmax(int num_layers, int64_t count, int in_dtype,
                 const void* const* k_in, uint32_t* max_bits, void* stream);

/*
 * pkv_decode — materialising read for `num_layers` layers in one launch.
 * Replaces kvpool.pool.AgentCacheView.get_kv_for_layer (pool.py:229-237):
 * dequantize_k (keyquant.py:68-71), dequantize_v (valuequant.py:222-238) and,
 * for out_dtype == PKV_BF16, round_to_bfloat16 (pool.py:66-76). Results are
 * bit-identical to the reference (bf16 output holds exactly the reference's
 * bf16-rounded f32 values). Either k_* or v_* arrays may be NULL.
 */
int pkv_decode(int num_layers, int64_t num_vectors, int head_dim, int out_dtype,
               int k_mode, const int8_t* const* k_codes,
               const float* const* k_scale, const uint16_t* const* k_bscale,
               const uint8_t* const* v_packed, const float* const* v_scales,
               const double* centroids_host, const uint32_t* sign_bits_host,
               void* const* k_out, void* const* v_out, void* stream);

/* Canonical uint8 codes <-> packed 3-bit payload over `count` codes
 * (valuequant.py:312-345). pkv_pack_codes ORs PKV_FLAG_BAD_CODE into
 * *bad_code (device uint32) when a code exceeds 7. */
int pkv_unpack_codes(const uint8_t* packed, int64_t count, uint8_t* codes,
                     void* stream);
int pkv_pack_codes(const uint8_t* codes, int64_t count, uint8_t* packed,
                   uint32_t* bad_code, void* stream);

/*
 * pkv_decode_attention — GQA decode attention that reads the packed pool
 * directly (no per-agent K/V copy). Replaces the eager/SDPA attention over a
 * materialised DynamicCache (transformers LlamaAttention.forward ->
 * eager_attention_forward, modeling_llama.py:199-230) for one layer.
 *
 *  q           [num_rows, kv_heads, group, head_dim] queries (f32 or bf16,
 *              `q_dtype`), num_rows = agents (one decode token each).
 *  pool        layer's K codes/scale and V packed/scales (prefix, T tokens).
 *  tail_k/v    optional per-row bf16 tail [num_rows, kv_heads, tail_cap,
 *              head_dim] holding tail_len[r] appended tokens (may be NULL).
 *  q_len       query positions per agent (1 for a decode step). With q_len
 *              > 1 (several new tokens per agent, e.g. a prompt suffix on top
 *              of the pool) the `group` rows of an agent are G * q_len, row
 *              g holds position g % q_len, and position i attends to the
 *              prefix plus the tail up to its own token (tail_len[r] counts
 *              all q_len new tokens): causal, no per-agent prefix copy.
 *  out         [num_rows, kv_heads, group, head_dim] f32 or bf16.
 *  softmax_scale  multiplier of q.k (head_dim**-0.5 for Llama).
 *  workspace   device scratch of pkv_attention_workspace_bytes(...).
 */
size_t pkv_attention_workspace_bytes(int num_rows, int kv_heads, int group,
                                     int head_dim, int64_t seq_len);
int pkv_decode_attention(int num_rows, int kv_heads, int group, int head_dim,
                         int64_t seq_len, int q_dtype, const void* q,
                         int k_mode, const int8_t* k_codes,
                         const float* k_scale, const uint16_t* k_bscale,
                         const uint8_t* v_packed, const float* v_scales,
                         const double* centroids_host,
                         const uint32_t* sign_bits_host,
                         const void* tail_k, const void* tail_v,
                         const int32_t* tail_len, int tail_cap, int q_len,
                         float softmax_scale, int out_dtype, void* out,
                         void* workspace, size_t workspace_bytes,
                         void* stream);

/*
 * pkv_layer_stats — build statistics of `num_layers` layers (LayerStats,
 * kvpool/pool.py:274-288, metrics.py:166-222) in one fused f64 reduction:
 * out[4*l + 0..3] = { sum (Kdec-K)^2, max |Kdec-K|, sum (Vdec-V)^2, sum V^2 }
 * over the `count` elements of layer l (double, device). k_in / v_in: the
 * source tensors (f32 or bf16, `in_dtype`); k_dec / v_dec: the f32 decode of
 * the pool (pkv_decode at PKV_F32 == the reference's 32-bit decode).
 * Deterministic (fixed reduction order). workspace: device scratch of
 * pkv_layer_stats_workspace_bytes(num_layers, count).
 */
size_t pkv_layer_stats_workspace_bytes(int num_layers, int64_t count);
int pkv_layer_stats(int num_layers, int64_t count, int in_dtype,
                    const void* const* k_in, const void* const* v_in,
                    const float* const* k_dec, const float* const* v_dec,
                    double* out, void* workspace, size_t workspace_bytes,
                    void* stream);

/* Internal self-checks that need the device. PKV_SELFTEST_DIVISION runs the
 * decode kernel's correctly-rounded x / f32(sqrt(d)) sequence for d in
 * {8, 32, 128} and the block32 key-scale x / 127 sequence against IEEE
 * division over every f32 mantissa; returns the number of mismatches
 * (0 expected) or a negative PKV_ERR_* code. Synchronises `stream`.
 * scratch: >= 16 bytes of device memory. */
#define PKV_SELFTEST_DIVISION 1
int64_t pkv_selftest(int what, void* scratch, size_t scratch_bytes, void* stream);

/* Host-side 64-bit FNV-1a over `n` bytes (kvpool/checksum.py:44-52). Used for
 * injection transcripts after a device->host copy; byte-serial by
 * definition, so it stays on the CPU. */
uint64_t pkv_fnv1a64(const void* data_host, size_t n);

/* FNV-1a of the little-endian f32 image of `count` bf16 values, without
 * materialising the f32 copy (== tensor_checksum(values.astype(f32))). */
uint64_t pkv_fnv1a64_bf16_as_f32(const uint16_t* data_host, size_t count);

#ifdef __cplusplus
}
#endif

#endif /* POLYKV_H_ */
