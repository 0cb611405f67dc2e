/* kvmix_b200.h -- C ABI of the B200-native TriAxialKV hot path (libkvmix_b200.so).
 *
 * Plain pointers and sizes only: no torch, no C++ types.  Every device pointer is
 * a CUDA device address; `stream` is a cudaStream_t (NULL = legacy default stream).
 * Every entry point is asynchronous on `stream` unless stated otherwise and returns
 * a status code; kvmix_last_error() gives the message of the last failure on the
 * calling thread.  Each entry point cites the reference (kvmix, /root/reference/pkg)
 * interface it replaces -- see INTEGRATION.md for the ctypes binding.
 *
 * Device pool layout, G = 32, d = head_dim:
 *   int2_pool : uint8 [L][Hkv][n_pages][page_stride(d) = 24 d]
 *               record = KeyPageBlock (d*G/4 + 4d B) + G INT2 V TokenBlocks (d/4 + 4d/G B each)
 *   int4_pool : uint8 [L][Hkv][n_int4][slot_stride(d)]
 *               record = INT4 K TokenBlock (d/2 + 4d/G B) + INT4 V TokenBlock, padded to 16 B
 * Every payload byte of every block (LAYOUT.md) is stored unmodified; inside a record the
 * bytes are permuted so each decode lane loads its MMA fragment with one wide load
 * (kvmix_page_layout / kvmix_slot_layout export the permutation).
 * Slot s < offset is INT2 page s/G row s%G; slot s >= offset is INT4 index s - offset.
 */
#ifndef KVMIX_B200_H
#define KVMIX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVMIX_GROUP_SIZE 32 /* quant.py:23 GROUP_SIZE */

/* status codes */
#define KVMIX_OK 0
#define KVMIX_EINVAL (-2)    /* reference ValidationError (errors.py:12) */
#define KVMIX_ECAPACITY (-3) /* reference CapacityError (errors.py:27) */
#define KVMIX_ECUDA (-5)     /* CUDA launch/runtime failure */

/* element types of float inputs/outputs */
#define KVMIX_F32 0
#define KVMIX_BF16 1
#define KVMIX_F16 2

const char* kvmix_version(void);
const char* kvmix_last_error(void);
/* cudaStreamSynchronize(stream) with the library's error reporting (used by the single-group
 * quantize / dequantize calls, which run one zero-copy kernel on pinned memory per call). */
int kvmix_stream_sync(void* stream);
/* record strides of the device pools (bytes) */
int64_t kvmix_page_stride(int64_t head_dim);
int64_t kvmix_slot_stride(int64_t head_dim);
/* Host-only (no GPU needed): perm[i] = byte of the reference-order record (KeyPageBlock ||
 * G INT2 V TokenBlocks, resp. INT4 K TokenBlock || INT4 V TokenBlock) stored at record byte i,
 * -1 for padding.  perm has page_stride(d) / slot_stride(d) entries. */
int kvmix_page_layout(int64_t head_dim, int64_t* perm);
int kvmix_slot_layout(int64_t head_dim, int64_t* perm);
/* payload sizes; replace quant.py:123-128 key_page_payload_bytes / token_block_payload_bytes */
int64_t kvmix_key_page_payload_bytes(int64_t head_dim);
int64_t kvmix_token_block_payload_bytes(int64_t head_dim, int64_t bitwidth);

/* ---- codec (K1) --------------------------------------------------------------- */

/* Replaces quant.py:160 encode_key_page_int2 (batched): keys f32 [n_pages][G][d] ->
 * out [n_pages][out_stride] with the KeyPageBlock payload at the start of each row.
 * err_flag (device int32, may be NULL) gets bit 0 set on non-finite input. */
int kvmix_encode_key_pages(const float* keys, int64_t n_pages, int64_t head_dim, uint8_t* out, int64_t out_stride,
                           int32_t* err_flag, void* stream);
/* Replaces quant.py:189 encode_token_block / :206 encode_token_blocks:
 * x f32 [n][d] -> out [n][out_stride], TokenBlock payload at the start of each row. */
int kvmix_encode_token_blocks(const float* x, int64_t n, int64_t head_dim, int32_t bitwidth, uint8_t* out,
                              int64_t out_stride, int32_t* err_flag, void* stream);
/* Replaces quant.py:180 decode_key_page_int2: blocks [n_pages][in_stride] -> f32 [n_pages][G][d] */
int kvmix_decode_key_pages(const uint8_t* blocks, int64_t n_pages, int64_t head_dim, int64_t in_stride, float* out,
                           void* stream);
/* Replaces quant.py:235 decode_token_blocks / :256 decode_token_block: [n][in_stride] -> f32 [n][d] */
int kvmix_decode_token_blocks(const uint8_t* blocks, int64_t n, int64_t head_dim, int32_t bitwidth,
                              int64_t in_stride, float* out, void* stream);
/* Replaces quant.py:64 quantize_group (batched, ragged): groups are x[offsets[i]:offsets[i+1]],
 * codes written at the same positions, scale/zero per group (fp32 holding the fp16 value). */
int kvmix_quantize_groups(const float* x, const int64_t* offsets, int64_t n_groups, int32_t bitwidth,
                          uint8_t* codes, float* scale, float* zero, int32_t* err_flag, void* stream);
/* Replaces quant.py:90 dequantize_group (batched, ragged): out = code * fp16(scale) + fp16(zero)
 * in fp32 (product and sum rounded separately); max_len = the longest group (grid size hint). */
int kvmix_dequantize_groups(const uint8_t* codes, const int64_t* offsets, int64_t n_groups, const float* scale,
                            const float* zero, float* out, int64_t max_len, void* stream);
/* Replaces quant.py:96 pack_codes / :112 unpack_codes. n codes <-> ceil(n*b/8) bytes.
 * pack sets err_flag bit 1 if a code is out of range. */
int kvmix_pack_codes(const uint8_t* codes, int64_t n, int32_t bitwidth, uint8_t* out, int32_t* err_flag,
                     void* stream);
int kvmix_unpack_codes(const uint8_t* packed, int64_t n, int32_t bitwidth, uint8_t* out, void* stream);

/* ---- pool data plane ------------------------------------------------------------- */

/* Pool status words (device int32[KVMIX_POOL_STATUS_WORDS], owned by the pool, zeroed at
 * creation): the pool writers (kvmix_write_prefill, kvmix_append_int4, the fused decode
 * append) set bit 0 of word ERR on non-finite input and raise KSCALE / VSCALE to the
 * largest INT2 key-page scale / V scale (INT2 and INT4) they stored, as fp32 bit patterns
 * (atomicMax; non-negative floats order like their bits).  The decode kernel reads the two
 * scales to bound its fp16 operands (q * s_k and p * s_v) without per-tile checks. */
#define KVMIX_POOL_STATUS_WORDS 4
#define KVMIX_POOL_STATUS_ERR 0
#define KVMIX_POOL_STATUS_KSCALE 1
#define KVMIX_POOL_STATUS_VSCALE 2

/* Replaces pool.py:228 MixedPrecisionPool.write_prefill (with write_page :201 and the INT4
 * branch :253-262): quantize+pack one request's prefill K/V [L][n_tokens][Hkv][d]
 * (dtype KVMIX_F32/BF16/F16, contiguous) into the pools.
 * page_tokens [n_req_pages][G]: token index of each page row (token order);
 * page_ids [n_req_pages]: destination page index; int4_tokens/int4_ids [n_req_int4].
 * err_flag: the pool status words (KVMIX_POOL_STATUS_*), may be NULL. */
int kvmix_write_prefill(const void* keys, const void* values, int32_t dtype, int64_t n_layers, int64_t n_tokens,
                        int64_t n_kv_heads, int64_t head_dim, const int32_t* page_tokens, const int32_t* page_ids,
                        int64_t n_req_pages, const int32_t* int4_tokens, const int32_t* int4_ids,
                        int64_t n_req_int4, uint8_t* int2_pool, int64_t pool_pages, uint8_t* int4_pool,
                        int64_t pool_int4, int32_t* err_flag, void* stream);

/* Replaces pool.py:284 append_decode_token (data half; the host pops the slot) and
 * pool.py:217 write_token: quantize n tokens' K/V [n][n_layers_in][Hkv][d] at INT4 into
 * int4 indices int4_ids[n], pool layers [layer0, layer0 + n_layers_in).
 * err_flag: the pool status words (KVMIX_POOL_STATUS_*), may be NULL. */
int kvmix_append_int4(const void* k, const void* v, int32_t dtype, int64_t n, int64_t n_layers_in, int64_t layer0,
                      int64_t n_layers, int64_t n_kv_heads, int64_t head_dim, const int32_t* int4_ids,
                      uint8_t* int4_pool, int64_t pool_int4, int32_t* err_flag, void* stream);
/* The same with explicit element strides of the input: element (token i, layer l, head h, channel c)
 * at k[l * layer_stride + i * tok_stride + h * head_dim + c] (kvmix_append_int4 is layer_stride =
 * n_kv_heads * head_dim, tok_stride = n_layers_in * n_kv_heads * head_dim; a layer-major step
 * buffer [n_layers_in][n][Hkv][d] is layer_stride = n * Hkv * d, tok_stride = Hkv * d). */
int kvmix_append_int4_strided(const void* k, const void* v, int32_t dtype, int64_t n, int64_t n_layers_in,
                              int64_t layer0, int64_t n_layers, int64_t n_kv_heads, int64_t head_dim,
                              int64_t layer_stride, int64_t tok_stride, const int32_t* int4_ids, uint8_t* int4_pool,
                              int64_t pool_int4, int32_t* err_flag, void* stream);

/* Replaces pool.py:394 PoolView.gather and pool.py:264 read_slot (K5): decode slots[m]
 * of one layer into k_out, v_out f32 [m][Hkv][d]. */
int kvmix_gather_dequant(const uint8_t* int2_pool, const uint8_t* int4_pool, int64_t pool_pages, int64_t pool_int4,
                         int64_t offset, int64_t layer, int64_t n_kv_heads, int64_t head_dim, const int32_t* slots,
                         int64_t m, float* k_out, float* v_out, void* stream);

/* K5 with a typed output: out_dtype KVMIX_F32 (== kvmix_gather_dequant), KVMIX_BF16 or KVMIX_F16
 * (round-to-nearest image of the exact dequantized value) -- the K/V of an fp16 / bf16
 * prefill attention over matched prefixes read straight from the pool. */
int kvmix_gather_dequant_typed(const uint8_t* int2_pool, const uint8_t* int4_pool, int64_t pool_pages,
                               int64_t pool_int4, int64_t offset, int64_t layer, int64_t n_kv_heads, int64_t head_dim,
                               const int32_t* slots, int64_t m, void* k_out, void* v_out, int32_t out_dtype,
                               void* stream);

/* ---- device-side page-table build (K6) ----------------------------------------------- */

/* Scratch size (int64 elements) of the routing counts for an n-token request. */
int64_t kvmix_route_scratch_elems(int64_t n);

/* Phase 1 of pool.py:122 alloc on the device: counts[0] = number of bitwidth-2 tokens of
 * bits[n] (int8, device), counts[1..] = per-chunk counts used by kvmix_route_tokens
 * (counts: device int64 [kvmix_route_scratch_elems(n)]).  Bits other than 2 / 4 set err bit 2.
 * The host reads counts[0] to pop its LIFO stacks (pool.py:131-148). */
int kvmix_count_int2(const int8_t* bits, int64_t n, int64_t* counts, int32_t* err_flag, void* stream);

/* Phase 2: replaces the O(N) token routing of pool.py:122-163 alloc and the index emission of
 * pool.py:228-262 write_prefill.  The host pops n_pages = counts[0] / page_size page starts and
 * n_int4 = n - n_pages * page_size INT4 slots (pop order) and passes them with the counts of
 * phase 1; the kernel writes
 *   slots[n]                       the PageTable (token order), identical to the host alloc
 *   page_tokens[n_pages][page_size], page_ids[n_pages]   K1 page inputs   (nullable)
 *   int4_tokens[n_int4], int4_ids[n_int4] (slot - offset) K1 INT4 inputs / K2 INT4 list (nullable)
 * The r-th INT2 token with r < n_pages * page_size gets page_starts[r / page_size] + r % page_size;
 * every other token takes the next INT4 pop in token order. */
int kvmix_route_tokens(const int8_t* bits, int64_t n, int32_t page_size, const int64_t* counts,
                       const int64_t* page_starts, int64_t n_pages, const int64_t* int4_pops, int64_t n_int4,
                       int64_t offset, int64_t* slots, int32_t* page_tokens, int32_t* page_ids,
                       int32_t* int4_tokens, int32_t* int4_ids, int32_t* err_flag, void* stream);

/* ---- decode attention (K2 + K3) ---------------------------------------------------- */

/* Replaces attention.py:175 flash_decode (+ PoolView.gather pool.py:394, _split_partial
 * attention.py:168, merge_partials attention.py:154), batched over requests, one layer,
 * one launch (the cross-split combine is fused into the kernel).
 *   q [batch][n_q_heads][d] (q_dtype), out [batch][n_q_heads][d] (out_dtype)
 *   page_indptr[batch+1], page_ids[]: INT2 page list of each partitioned table (table order)
 *   int4_indptr[batch+1], int4_ids[]: INT4 indices of each table's suffix (table order)
 *   int4_count: NULL for CSR lists; else request b's INT4 list is int4_ids[int4_indptr[b] ..
 *     int4_indptr[b] + int4_count[b]) (the padded lists kept by kvmix_decode_tables)
 *   The tiles of a unit (request b, kv head h; unit = b*Hkv + h) are its INT2 pages then
 *   ceil(n_int4/32) INT4 tiles of 32 slots, so every tile is bitwidth-homogeneous.
 *   work [n_pieces][8] = {unit, tile_lo, tile_hi, slot, part0, nparts, 0, 0}: a piece is a
 *     contiguous tile range of one unit; slot = -1 if the piece is the whole unit, else its
 *     partial slot in partials [n_parts][8][d + 4], the unit's partials being slots
 *     part0 .. part0 + nparts - 1.
 *   cta_ptr [n_cta + 1]: CTA i runs pieces cta_ptr[i] .. cta_ptr[i+1] (a byte-balanced share
 *     of the batch, see plan.py); the last CTA to finish a split unit merges its partials.
 *   counters [batch * Hkv] int32, zero before the first launch; every launch leaves them zero.
 *   variant: 0 = tensor-core kernel (mma.sync m16n8k16; plan with 3 CTAs per SM), 1 = simple
 *     CUDA-core kernel (fp32-faithful); measurement builds (-DKVMIX_MEASURE_VARIANTS) add
 *     2 = data movement only, 3 = compute only on stale smem (output meaningless)
 *   pool_status: the pool status words (KVMIX_POOL_STATUS_*); NULL = operand bounds unknown
 *     (exact-max softmax and q pre-scaled for the largest finite scales: correct, slower).
 *   flags: KVMIX_DECODE_POOL_WRITTEN when a kernel that wrote this pool (write_prefill,
 *     append_int4, ...) precedes the launch in the stream: the kernel then waits for it before
 *     its first KV copies (otherwise they overlap the previous kernel's tail through
 *     programmatic dependent launch).
 * Requires n_q_heads % Hkv == 0 and n_q_heads / Hkv <= 8, d in {32, 64, 128}. */
#define KVMIX_DECODE_POOL_WRITTEN 1
int kvmix_flash_decode(const void* q, int32_t q_dtype, void* out, int32_t out_dtype, const uint8_t* int2_pool,
                       const uint8_t* int4_pool, int64_t pool_pages, int64_t pool_int4, int64_t layer,
                       int64_t n_kv_heads, int64_t head_dim, int64_t n_q_heads, int64_t batch,
                       const int32_t* page_indptr, const int32_t* page_ids, const int32_t* int4_indptr,
                       const int32_t* int4_ids, const int32_t* int4_count, const int32_t* work,
                       const int32_t* cta_ptr, int64_t n_cta, float* partials, int32_t* counters, float scale,
                       int32_t variant, int32_t* pool_status, int32_t flags, void* stream);

/* KV-head-parallel combine fused into the decode (cfg4; the all-gather of pool.py:108-110's
 * head-agnostic slots + attention.py:198-201's kv = h // ratio): identical to kvmix_flash_decode,
 * except that this rank's n_q_heads output heads are stored at head offset out_head0 of each of
 * the n_outs (1..8) buffers outs[] = [batch][out_heads][d] (out_dtype): device addresses this
 * process can store to -- its own gathered output and the peers' ones mapped over NVLink (e.g.
 * torch symmetric memory).  The kernel's epilogue stores every finished head slice straight into
 * every rank's buffer, so no separate all-gather runs; the caller orders the peers' reads after
 * all ranks' launches (a symmetric-memory barrier).  outs is a HOST array of device addresses. */
int kvmix_flash_decode_gather(const void* q, int32_t q_dtype, void* const* outs, int32_t n_outs, int64_t out_heads,
                              int64_t out_head0, int32_t out_dtype, const uint8_t* int2_pool, const uint8_t* int4_pool,
                              int64_t pool_pages, int64_t pool_int4, int64_t layer, int64_t n_kv_heads,
                              int64_t head_dim, int64_t n_q_heads, int64_t batch, const int32_t* page_indptr,
                              const int32_t* page_ids, const int32_t* int4_indptr, const int32_t* int4_ids,
                              const int32_t* int4_count, const int32_t* work, const int32_t* cta_ptr, int64_t n_cta,
                              float* partials, int32_t* counters, float scale, int32_t variant, int32_t* pool_status,
                              int32_t flags, void* stream);

/* K4 fused decode append (pool.py:284-306 append_decode_token data half + attention.py:175
 * flash_decode, one launch): the same as kvmix_flash_decode (variant 0) for one layer, where
 * the host has already popped one INT4 slot per request and appended it to the table (the
 * last entry of int4_ids of each request).  The warp that owns that slot's tile quantizes
 * k_new / v_new [batch][n_kv_heads][d] (kv_dtype) into the tile it is about to read and into
 * int4_pool, so the new token is both stored and attended to. */
int kvmix_flash_decode_append(const void* q, int32_t q_dtype, void* out, int32_t out_dtype, uint8_t* int2_pool,
                              uint8_t* int4_pool, int64_t pool_pages, int64_t pool_int4, int64_t layer,
                              int64_t n_kv_heads, int64_t head_dim, int64_t n_q_heads, int64_t batch,
                              const int32_t* page_indptr, const int32_t* page_ids, const int32_t* int4_indptr,
                              const int32_t* int4_ids, const int32_t* int4_count, const int32_t* work,
                              const int32_t* cta_ptr, int64_t n_cta, float* partials, int32_t* counters, float scale,
                              const void* k_new, const void* v_new, int32_t kv_dtype, int32_t* pool_status,
                              int32_t flags, void* stream);

/* K7 decode-step tables (pool.py:284-306 append_decode_token, the device half): append
 * new_slots[b] (INT4 index = slot - offset; NULL = no append) to request b's padded INT4
 * list int4_ids[b * cap + int4_count[b]] and bump int4_count[b] (err bit 2 when full), then
 * rebuild the decode kernel's stream-K plan for n_pages[b] INT2 pages and int4_count[b]
 * INT4 slots per request: work [n_cta + batch * n_kv][8] (capacity), cta_ptr [n_cta + 1],
 * n_parts [1] (partial slots used, <= n_cta + batch * n_kv), scratch int32 [2 * batch * n_kv].
 * Use with kvmix_flash_decode(_append)(int4_indptr[b] = b * cap, int4_count, ...). */
int64_t kvmix_decode_tables_smem(int64_t batch, int64_t n_cta);
int kvmix_decode_tables(const int32_t* new_slots, int64_t batch, int64_t n_kv, const int32_t* n_pages,
                        int32_t* int4_count, int32_t* int4_ids, int64_t cap, int64_t head_dim, float int4_weight,
                        int64_t n_cta, int32_t* work, int32_t* cta_ptr, int32_t* n_parts, int32_t* scratch,
                        int32_t* err, void* stream);

/* Replaces attention.py:32 attention_full (the calibration replay's dense attention, used by
 * calibration.py:108-125 measure_raw): q f32 [n_q][n_heads][d], k / v f32 [n_k][n_kv_heads][d],
 * out f32 [n_q][n_heads][d]; causal aligns the queries to the last n_q keys.  fp32, d in {32, 64, 128, 256}. */
int kvmix_attention_full(const float* q, const float* k, const float* v, int64_t n_q, int64_t n_k, int64_t n_heads,
                         int64_t n_kv_heads, int64_t head_dim, float scale, int32_t causal, float* out, void* stream);
/* Replaces attention.py:154 merge_partials for explicit partials (natural-log domain):
 * acc [n][d], lse [n], max_logit [n] (device f32) -> out [d]. n >= 1. */
int kvmix_merge_partials(const float* acc, const float* lse, const float* max_logit, int64_t n, int64_t d, float* out,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KVMIX_B200_H */
