/*
 * tsv.h -- C ABI of the B200-native TurboSpec propose / verify / accept step.
 *
 * TurboSpec (arXiv 2406.14066): one speculative-decoding step is
 *   GetProposedLen / Propose -> GetVerificationLen -> Score -> Accept ->
 *   UpdateGlobalAcceptance                          (Listing 1)
 * This library implements the data-parallel parts of that step on sm_100a:
 *   tsv_propose_lookup     prompt-lookup n-gram proposal
 *   tsv_goodput_choose_k   ArgMaxGoodput over k = 0..K          (Listing 2)
 *   tsv_verify_accept      rejection-sampling acceptance + bonus
 *   tsv_update_acceptance  moving-average acceptance update
 * The target model's Score step is not here: its output (probability rows p)
 * is an input.  Readings of silent or garbled passages are numbered R1..R26
 * in DESIGN.md section 3 and cited below.  Beyond the four calls: vocab-
 * sharded and request-sharded variants (NCCL), greedy and softmax-from-logits
 * verify, a fused verify + update, and a closed-loop harness.
 *
 * Conventions (all entry points):
 *  - Array arguments are DEVICE-ACCESSIBLE pointers owned by the caller; the
 *    library never allocates, frees or retains them.  Read-only inputs may also
 *    live in pinned host memory (cudaHostAlloc / torch pin_memory(), mapped
 *    into the device address space by UVA): the kernels then read exactly the
 *    bytes they need over PCIe (zero-copy; e.g. only row m of p and q in the
 *    lazy verify).  Outputs and workspaces must be device memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is asynchronous on `stream`, never synchronises, never
 *    allocates device memory, and is CUDA-graph capturable.
 *  - Host-side argument validation happens before any launch; a non-OK status
 *    means nothing was launched.  tsv_last_error() returns a thread-local
 *    message for the last non-OK status of the calling thread.
 *  - Data errors that can only be seen on the device (token id out of range,
 *    ragged offsets decreasing or reaching past rows_p / the draft rows,
 *    k_i > k_max, a context longer than TSV_MAX_CONTEXT) never trap and
 *    never touch memory outside the caller's arrays: the affected request's
 *    outputs are -1 and, when `device_status` is non-NULL, the matching
 *    TSV_DEVSTATUS_* bit is OR-ed into *device_status.
 *  - Workspaces: a NULL or too small workspace / scratch returns
 *    TSV_ERR_WORKSPACE (nothing launched).
 *  - Results are a pure function of (inputs, seed, step, request_ids): they do
 *    not depend on grid size, chunking, vocab sharding, batch order or stream.
 *  - Floating point: no fast-math, no FTZ; IEEE binary32 for probabilities
 *    and race scores, binary64 for the goodput model; explicit FMAs only.
 *  - Only sm_100 (B200) devices are accepted (TSV_ERR_UNSUPPORTED_DEVICE).
 */
#ifndef TSV_H
#define TSV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSV_ABI_VERSION 2  /* 2: device_status on the lookups, step_counts in tsv_verify_args */

#if defined(__GNUC__)
#define TSV_API __attribute__((visibility("default")))
#else
#define TSV_API
#endif

typedef enum {
    TSV_OK = 0,
    TSV_ERR_INVALID_ARG = 1,        /* bad host argument; nothing launched          */
    TSV_ERR_CUDA = 2,               /* a CUDA runtime call failed                   */
    TSV_ERR_NCCL = 3,               /* NCCL unavailable or an NCCL call failed      */
    TSV_ERR_UNSUPPORTED_DEVICE = 4, /* current device is not sm_100                 */
    TSV_ERR_WORKSPACE = 5           /* workspace / scratch NULL or smaller than     */
                                    /* required (its *_workspace_size call)         */
} tsv_status;

/* bits OR-ed into *device_status by the kernels */
#define TSV_DEVSTATUS_BAD_TOKEN 1u  /* draft token outside [0, vocab_global)      */
#define TSV_DEVSTATUS_BAD_K 2u      /* k_i < 0 or k_i > k_max (ragged offsets)    */
#define TSV_DEVSTATUS_NO_WEIGHT 4u  /* selected p row has no positive entry        */
#define TSV_DEVSTATUS_P2P_TIMEOUT 8u /* a peer-memory exchange wait gave up (a peer
                                        never arrived); outputs are not valid      */
#define TSV_DEVSTATUS_WAIT_TIMEOUT 32u /* a bounded wait for alpha_ready gave up (its
                                           producer never ran: a contract violation) */
#define TSV_DEVSTATUS_BAD_CONTEXT 16u /* lookup: ctx_offsets negative or decreasing,
                                          or L_i > TSV_MAX_CONTEXT                 */

TSV_API const char* tsv_last_error(void);
TSV_API int tsv_abi_version(void);

/* --------------------------------------------------------------------------
 * Prompt-lookup proposal (PLD).  PAPER.md:57 [AD] "We use a fixed-length
 * proposal strategy ... each request attempts to retrieve a predetermined
 * number of tokens ... the proposal cost only depends on the context search";
 * PAPER.md:454 "proposed tokens are retrieved as n-grams from the input
 * prompt"; Fig. PAPER.md:44-49 (a request without a match proposes nothing).
 * Reading R20: for n = n_max down to n_min, the latest start s < L-n with
 * ctx[s..s+n-1] == ctx[L-n..L-1] (self-match excluded, overlap allowed);
 * propose ctx[s+n .. min(s+n+k_fixed, L)-1]; no match => length 0.
 *   ctx          int32 [ctx_offsets[B]]  token ids, requests concatenated
 *   ctx_offsets  int32 [B+1]             request i owns ctx[off[i] .. off[i+1]);
 *                                        L_i = off[i+1]-off[i] <= TSV_MAX_CONTEXT
 *   n_min,n_max  1 <= n_min <= n_max <= TSV_MAX_NGRAM
 *   k_fixed      FIXED_PROPOSED_LEN, 1..TSV_MAX_K (Listing 1 line 26)
 *   proposals    int32 [B, k_fixed] out, -1 padded
 *   proposal_len int32 [B] out (0..k_fixed)
 *   device_status int32 [1] nullable; TSV_DEVSTATUS_BAD_CONTEXT is OR-ed in for a
 *                request whose offsets are negative / decreasing or whose L_i >
 *                TSV_MAX_CONTEXT (the kernel packs the end position in 20 bits);
 *                that request proposes nothing (length 0, all -1)
 * Errors: INVALID_ARG for B < 0, bad n/k range, NULL arrays (B > 0).
 * ------------------------------------------------------------------------ */
#define TSV_MAX_CONTEXT (1 << 20)
#define TSV_MAX_NGRAM 64
#define TSV_MAX_K 15

TSV_API tsv_status tsv_propose_lookup(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                              int32_t n_min, int32_t n_max, int32_t k_fixed,
                              int32_t* proposals, int32_t* proposal_len, int32_t* device_status,
                              void* stream);

/* tsv_propose_lookup with flags (tsv_propose_lookup == flags 0).
 *   TSV_LOOKUP_INPUTS_READY  Contract: no kernel that can still be in flight
 *     when this call's kernel starts writes its inputs (ctx, ctx_offsets) or
 *     reads its outputs (proposals, proposal_len).  Under programmatic
 *     dependent launch a kernel may start while its predecessor drains; every
 *     libtsv kernel triggers its dependents only after its own grid-dependency
 *     wait, so in a chain of libtsv calls only the IMMEDIATELY preceding kernel
 *     can be in flight (data written two or more kernels back is complete), and
 *     a kernel launched without programmatic serialization is complete.  True
 *     e.g. when the context buffer is prepared before the step (a serving
 *     engine's input preparation); NOT when the immediately preceding kernel
 *     appends to it.  The whole lookup then runs before the grid-dependency
 *     wait, overlapping the preceding kernel; the kernel waits at its end (it
 *     still completes after its predecessor).  Outputs identical to flags 0.
 * Errors: as tsv_propose_lookup; INVALID_ARG for unknown flags. */
#define TSV_LOOKUP_INPUTS_READY 1
TSV_API tsv_status tsv_propose_lookup_ex(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                                 int32_t n_min, int32_t n_max, int32_t k_fixed,
                                 int32_t* proposals, int32_t* proposal_len, int32_t* device_status,
                                 int32_t flags, void* stream);

/* --------------------------------------------------------------------------
 * Verify / accept.  PAPER.md:18 [AD] "we utilize rejection sampling to
 * determine which tokens are retained ... (2) a bonus token that either
 * rectifies an incorrect draft prediction or extends the sequence when all
 * proposed tokens are accepted"; PAPER.md:493-497 [BG] (k+1 target
 * distributions; m+1 tokens, minimum 1, maximum k+1; zero accuracy loss).
 * Per request i (k_i drafts x_j, target rows p_0..p_k, draft rows q_0..q_{k-1}):
 *   m = first j with !(RN32(u_acc(i,j) * q_j[x_j]) < p_j[x_j]), else k   (R1-R4)
 *   w = m < k ? max(0, RN32(p_m - q_m)) : max(0, p_k); all-zero w -> p_m (R5)
 *   t = argmax_v RN32(w_v / E(u_race(i,m,v))), lowest v on ties     (R7-R9)
 *   out_tokens[i] = (x_0 .. x_{m-1}, t, -1 ...); num_accepted[i] = m
 * Uniforms: Philox4x32-10 keyed by seed, counter (v>>2, purpose<<16|pos,
 * request_id, step) with GLOBAL vocab index and GLOBAL request id (R6).
 *
 * Layout: p is [rows_p, ld] fp32 row-major with 16-byte aligned rows
 * (ld % 4 == 0, base 16-byte aligned); request i owns p rows
 * row_offsets[i] .. row_offsets[i+1]-1 (k_i + 1 rows, so
 * k_i = row_offsets[i+1]-row_offsets[i]-1).  q (NULL => one-hot drafts, e.g.
 * PLD / top-1) is [rows_p - B, ld] with request i's rows and drafts at
 * row_offsets[i]-i .. +k_i-1 (same packing as draft_tokens).  Only columns
 * [0, vocab) of each row are read (the allocation must still cover
 * round-up-to-4(vocab) columns, which ld % 4 == 0 guarantees).
 * Vocab shards: local column c is global index vocab_offset + c
 * (vocab_offset % 4 == 0); draft ids are global.
 * ------------------------------------------------------------------------ */
typedef struct tsv_verify_args {
    const float* p;               /* [rows_p, ld]                                  */
    const float* q;               /* [rows_p - B, ld] or NULL (one-hot drafts)      */
    const int32_t* row_offsets;   /* [B+1]                                          */
    const int32_t* draft_tokens;  /* [rows_p - B], global ids                       */
    const uint32_t* request_ids;  /* [B] global request ids (Philox stream)         */
    int32_t* num_accepted;        /* [B] out (m_i; -1 on a data error)              */
    int32_t* out_tokens;          /* [B, k_max+1] out, -1 padded                    */
    int32_t* device_status;       /* nullable; TSV_DEVSTATUS_* bits OR-ed in        */
    void* workspace;              /* see tsv_verify_workspace_size                  */
    uint64_t workspace_bytes;
    int64_t ld;                   /* row stride in elements, % 4 == 0               */
    uint64_t seed;                /* Philox key                                     */
    uint32_t step;                /* Philox counter word 3 (decode step)            */
    int32_t B;                    /* requests                                       */
    int32_t k_max;                /* 0..TSV_MAX_K; out_tokens row length k_max+1    */
    int32_t rows_p;               /* sum_i (k_i + 1); host-known size of p          */
    int32_t vocab;                /* local columns in this shard (>= 1)             */
    int32_t vocab_offset;         /* global index of local column 0 (% 4 == 0)      */
    int32_t vocab_global;         /* global vocabulary size                         */
    int32_t chunk;                /* 0 = auto (~1 item per resident warp); else     */
                                  /* vocab columns per work item, a multiple of 128 */
                                  /* up to 16384: a tuning / test knob that never   */
                                  /* changes results                                */
    int32_t flags;                /* TSV_VERIFY_* bits                              */
    int64_t* step_counts;         /* nullable, device [2] out: (sum_i m_i, sum_i     */
                                  /* tested_i) over the valid requests, tested_i =  */
                                  /* m_i + [m_i < k_i] -- the per-step numerator and */
                                  /* denominator of the acceptance-rate estimate    */
                                  /* (R18); written by every verify */
                                  /* flavour (lazy, greedy, logits, sharded)        */
} tsv_verify_args;

#define TSV_VERIFY_NO_PRUNE 1     /* evaluate every race element exactly (test)     */
#define TSV_VERIFY_SHARD_DENSE 2  /* tsv_verify_accept_sharded: one-round dense mode  */
#define TSV_VERIFY_RACE_ONLY 4    /* measurement only (tsv_verify_accept): launch the */
                                  /* race kernel alone over the workspace left by a  */
                                  /* previous call with identical arguments; the race */
                                  /* max-combines into the same row keys, so outputs  */
                                  /* are unchanged.  bench.py times the dominant     */
                                  /* kernel with it.                                  */
#define TSV_VERIFY_P2P_FUSED 16   /* tsv_verify_accept_sharded_p2p / _phase: the race */
                                  /* kernel's work items push their chunk keys to     */
                                  /* every rank themselves (LL lines, no keys kernel);*/
                                  /* every rank must pass it; each shard must fit the */
                                  /* NC chunk slots sized for ceil4(vocab_global /    */
                                  /* world) columns (INVALID_ARG otherwise)           */
#define TSV_VERIFY_EARLY_TRIGGER 32 /* tsv_verify_accept / _update: the emit kernel  */
                                  /* lets the kernel after the call launch (PDL)      */
                                  /* before the race completes, so that kernel's CTAs */
                                  /* run in the SM slots the race's tail frees.       */
                                  /* Contract: the kernel after the call reads        */
                                  /* nothing the call writes (num_accepted,           */
                                  /* out_tokens, alpha, step_counts, device_status,   */
                                  /* the workspace) before its own grid-dependency    */
                                  /* wait -- true of every libtsv kernel without a    */
                                  /* *_READY flag, and of a TSV_LOOKUP_INPUTS_READY   */
                                  /* lookup whose contexts this call does not write.  */
                                  /* With it, two kernels of this call (race, emit)   */
                                  /* can be in flight when the next kernel starts.    */
                                  /* Outputs are unchanged.                           */
#define TSV_VERIFY_META_READY 8   /* Contract: row_offsets, draft_tokens and          */
                                  /* request_ids are COMPLETE before the kernel that  */
                                  /* immediately precedes this call on the stream     */
                                  /* could start, i.e. no kernel still in flight when */
                                  /* this call's first kernel launches writes them    */
                                  /* (e.g. they come from the proposer, before the    */
                                  /* target forward).  Under PDL a kernel may launch  */
                                  /* while its predecessor drains, so "not written by */
                                  /* the preceding kernel" is not enough if that      */
                                  /* kernel itself triggered early.  The scan then    */
                                  /* reads them before its grid-dependency wait and   */
                                  /* waits only before reading p and q (it prefetches */
                                  /* the p / q words it will gather into L2 before    */
                                  /* the wait: no data is read, L2 is coherent for    */
                                  /* writes).  Honoured by                            */
                                  /* tsv_verify_accept and tsv_verify_accept_update;  */
                                  /* ignored by every other entry point (sharded,     */
                                  /* greedy, logits).  libtsv's own kernels trigger   */
                                  /* their dependents only after their own wait.      */

/* Workspace: device scratch for per-request scan results and per-chunk race
 * keys (size from tsv_verify_workspace_size; no initialisation needed).  One
 * workspace per stream: concurrent calls must not share it. */
TSV_API tsv_status tsv_verify_workspace_size(const tsv_verify_args* a, size_t* bytes);
TSV_API tsv_status tsv_workspace_clear(void* workspace, size_t bytes, void* stream);
TSV_API tsv_status tsv_verify_accept(const tsv_verify_args* a, void* stream);

/* Greedy (temperature-0) verify, reading R24 (SURVEY.md
 * 8(f) NEXT(2)): keep draft j iff x_j = argmax_v p_j[v] (first maximum, NaN never
 * selected), emit the argmax of row m (correction at the first mismatch, or the
 * bonus after k accepted drafts).  Same arguments as tsv_verify_accept; q, seed,
 * step and request_ids are not used (request_ids may be NULL); vocab_offset must be
 * 0.  Streams every p row of the batch (each needs its full argmax).  Outputs and
 * device_status exactly as tsv_verify_accept (NO_WEIGHT: an all-NaN row). */
TSV_API tsv_status tsv_verify_greedy(const tsv_verify_args* a, void* stream);

/* Fused softmax-from-logits verify, reading R23: a->p and
 * a->q hold LOGITS (same layout as the probability rows; q may be NULL for one-hot
 * drafts).  Per row p_v = RN32(expf(RN32(RN32(z_v - M) * RN32(1/temperature))) *
 * RN32(1/S)), M = max z, S = binary64 sum of the exponentials; then exactly the
 * verify of tsv_verify_accept on those probabilities.  The probabilities are never
 * written: one dense pass over every p and q row of the batch computes per-chunk
 * online softmax partials, the acceptance scan combines them per tested row, and the
 * lazy race forms row m's probabilities from its logits while streaming it.
 * Parity with the CPU oracle is within 1e-6 relative on probabilities (CUDA expf is
 * within 2 ulp, the sums are reordered); decisions inside that margin may flip.
 * Workspace: tsv_verify_logits_workspace_size (zero-filled not required).
 * tsv_softmax_rows: the same probabilities written out for `rows` rows of z
 * (fp32 [rows, ld]; columns >= vocab of p_out are set to 0). */
TSV_API tsv_status tsv_verify_logits_workspace_size(const tsv_verify_args* a, size_t* bytes);
TSV_API tsv_status tsv_verify_accept_logits(const tsv_verify_args* a, float temperature, void* stream);
TSV_API tsv_status tsv_softmax_rows(const float* z, int64_t ld, int32_t vocab, int32_t rows, float temperature,
                                    float* p_out, void* stream);

/* Vocab-sharded verify (the target's LM head split over G ranks as under
 * tensor parallelism).  Rank g holds columns
 * [vocab_offset, vocab_offset + vocab) of every p and q row.
 *  partial: one round, dense over all rows of every request; writes one
 *           tsv_shard_tuple per p row (local packed argmax keys + the accept
 *           flag of draft tokens this shard owns);
 *  combine: given the G ranks' tuple arrays concatenated ([G][rows_p]), forms
 *           m_i (OR of flags, first-rejection scan), the winning key (max over
 *           ranks; the fallback key when the residual was zero everywhere) and
 *           writes num_accepted / out_tokens exactly as tsv_verify_accept.
 * Between them the caller exchanges tuples (NCCL all-gather, or loopback on
 * one device); tsv_verify_accept_sharded does all three with a tsv_comm. */
typedef struct tsv_shard_tuple {
    uint64_t key;      /* (bits(score) << 32) | (0xFFFFFFFF - global_v); 0 = none */
    uint64_t fb_key;   /* same over max(0, p_m) when the local residual is all 0   */
    uint32_t flag;     /* bit0: accept (owner of x_j only), bit1: owner,          */
                       /* bits 8..: TSV_DEVSTATUS_* seen by this shard             */
    uint32_t pad;
} tsv_shard_tuple;

TSV_API tsv_status tsv_verify_shard_partial(const tsv_verify_args* a, tsv_shard_tuple* tuples_out,
                                    void* stream);
TSV_API tsv_status tsv_verify_shard_combine(const tsv_verify_args* a, const tsv_shard_tuple* gathered,
                                    int32_t num_shards, void* stream);

/* Lazy two-round vocab sharding (SURVEY.md 8(e) variant; the default of
 * tsv_verify_accept_sharded): each rank streams only the selected row m_i of
 * its columns (about 1.6 rows per request at alpha = 0.7 instead of 2k+1).
 *  flags: masks_out[i] (uint64, device [B]) = (owner bits << 32) | accept bits
 *         of the drafts x_j (j < k_i) whose column this shard holds.  Owners
 *         are disjoint, so the integer SUM of the ranks' words is their OR.
 *  race:  from the summed masks (identical on every rank) forms m_i (first
 *         rejection; a draft owned by no shard makes the request bad), races
 *         row m_i over this shard's columns and writes keys_out[2i] = local
 *         packed key, keys_out[2i+1] = local fallback key (only when the local
 *         residual is all zero); device [2B].  Needs the verify workspace.
 *  emit:  from the summed masks and the element-wise MAX of the ranks' keys,
 *         writes num_accepted / out_tokens / device_status exactly as
 *         tsv_verify_accept.
 * Exchanges: ncclAllReduce(sum, uint64, B) after flags, ncclAllReduce(max,
 * uint64, 2B) after race (or any exact sum / max, e.g. loopback). */
TSV_API tsv_status tsv_verify_shard_flags(const tsv_verify_args* a, uint64_t* masks_out, void* stream);
TSV_API tsv_status tsv_verify_shard_race(const tsv_verify_args* a, const uint64_t* masks, uint64_t* keys_out,
                                         void* stream);
TSV_API tsv_status tsv_verify_shard_emit(const tsv_verify_args* a, const uint64_t* masks, const uint64_t* keys,
                                         void* stream);

/* Lazy two-round vocab sharding over NVLink peer memory:
 * the same computation as tsv_verify_accept_sharded's lazy mode, with both exchanges
 * done by the producing kernels themselves instead of NCCL all-reduces.  Every rank
 * owns one symmetric buffer (tsv_p2p_alloc, zero-filled; B_max requests), mapped
 * into every peer (tsv_p2p_open of the 64-byte CUDA IPC handle; the caller exchanges
 * handles, e.g. torch.distributed all_gather_object).  Every exchanged 32-bit word
 * travels with the call's epoch in one aligned 8-byte word {data, epoch}, stored
 * with 16-byte vector stores into slot [rank] of every peer's buffer; the consumer
 * polls its own buffer until each word carries the epoch (no fences, no grid
 * barrier).  Round 1: the flags kernel pushes the mask words, the meta kernel sums
 * the G slots (disjoint owners: the sum is the OR).  Round 2: the keys kernel pushes
 * the (key, fallback key) pairs after the race, the emit kernel takes their max.
 * Slots alternate by epoch parity.  A wait that never completes (a peer died) gives
 * up after seconds and sets TSV_DEVSTATUS_P2P_TIMEOUT instead of hanging.
 *  tsv_p2p_init: bufs[g] = rank g's buffer as mapped in this process (bufs[rank]
 *    local), world <= TSV_P2P_MAX_WORLD, B <= B_max in every call.  The call epoch
 *    is kept on the device (advanced by the emit kernel), so the calls can be
 *    captured in CUDA graphs; all ranks must make the same sequence of calls.
 *  tsv_verify_accept_sharded_p2p: the whole step on `stream` (flags -> meta -> race
 *    -> keys -> emit, five kernels, no host synchronisation); needs the verify
 *    workspace (tsv_verify_workspace_size).
 *  tsv_verify_shard_p2p_phase: phase 0 (flags + push), 1 (wait, meta, race, keys +
 *    push), 2 (wait, emit) separately: lets one process drive G loopback ranks on
 *    one device (all phase 0, then all 1, then all 2).
 *  flags & TSV_VERIFY_P2P_FUSED (every rank): no keys kernel -- each race work item
 *    (request i, chunk c) pushes its chunk key as one LL line into slot [rank][c][i]
 *    of every rank's buffer and the emit takes the max over the G x NC lines (NC:
 *    chunk slots per rank, the same on every rank, from vocab_global, world, B and
 *    the SM count); an item whose chunk has no positive residual pushes its share of
 *    the R5 fallback instead (flagged in bit 63).  Four kernels per call; outputs
 *    identical to the LL keys kernel. */
#define TSV_P2P_MAX_WORLD 8
#define TSV_P2P_MAX_SUMS 64
typedef struct tsv_p2p tsv_p2p;
TSV_API tsv_status tsv_p2p_buffer_size(int32_t B_max, size_t* bytes);
TSV_API tsv_status tsv_p2p_alloc(int32_t B_max, void** buf_out, void* ipc_handle_out /* 64 B, nullable */);
TSV_API tsv_status tsv_p2p_free(void* buf);
TSV_API tsv_status tsv_p2p_open(const void* ipc_handle /* 64 B */, void** buf_out);
TSV_API tsv_status tsv_p2p_close(void* buf);
TSV_API tsv_status tsv_p2p_init(tsv_p2p** out, int32_t rank, int32_t world, int32_t B_max, void* const* bufs);
TSV_API tsv_status tsv_p2p_destroy(tsv_p2p* p);
TSV_API tsv_status tsv_verify_accept_sharded_p2p(const tsv_verify_args* a, tsv_p2p* p, void* stream);
TSV_API tsv_status tsv_verify_shard_p2p_phase(const tsv_verify_args* a, tsv_p2p* p, int32_t phase, void* stream);
/* tsv_allreduce_i64_p2p: in-place exact sum over the ranks of count <= TSV_P2P_MAX_SUMS
 * int64 (device) through the same buffers (one CTA; LL words; its own device epoch), the
 * peer-memory replacement of tsv_allreduce_i64 for the request-sharded global sums
 * (tsv_goodput_partial -> this -> tsv_goodput_finalize; tsv_update_partial -> this ->
 * tsv_update_finalize).  device_status (nullable) gets TSV_DEVSTATUS_P2P_TIMEOUT. */
TSV_API tsv_status tsv_allreduce_i64_p2p(int64_t* data, int32_t count, tsv_p2p* p, int32_t* device_status,
                                         void* stream);

/* --------------------------------------------------------------------------
 * Goodput k selection: ArgMaxGoodput (Listing 2) over
 * k = 0..k_max (R12), Goodput = generated tokens / execution time (Eq.
 * goodput PAPER.md:38-42), generated tokens = sum_i l(alpha_i, k_i) with
 * l(a,k) = (1-a^{k+1})/(1-a) (Eq. gen_len) evaluated by
 * Horner, k_i = min(k, cap_i) (R13), time = T_target + T_draft (Eq.
 * batch-latency PAPER.md:103) with T_fwd = a*N_ctx + gamma*N_batched + delta
 * (Eq. forward-time), T_draft = k * T_fwd^draft (PAPER.md:128,
 * R15) or pld_cost_ms (R16).  Skips k > 0 with sum_i (k_i+1) > kv_free_slots
 * (OOM, R14); strict '>' keeps the smaller k on ties.
 *   alpha       fp64 [B] (alpha_per_request != 0) or [1]
 *   ctx_len     int32 [B] context tokens of each request (N_context terms)
 *   cap         int32 [B] per-request proposal cap (k_max for the draft
 *               policy; the PLD proposal length for TSV_POLICY_PLD, R21)
 *   k_out       int32 [1] out: k*
 *   goodput_out fp64 [k_max+1] out (nullable): tokens per ms, -1 for OOM k
 *   k_per_request int32 [B] out (nullable): min(k*, cap_i)
 * ------------------------------------------------------------------------ */
typedef struct tsv_latency_model {
    double ctx_ms_per_tok;      /* paper's alpha in Eq. forward-time            */
    double batched_ms_per_tok;  /* gamma                                        */
    double fixed_ms;            /* delta                                        */
} tsv_latency_model;

#define TSV_POLICY_DRAFT 0
#define TSV_POLICY_PLD 1

TSV_API tsv_status tsv_goodput_choose_k(const double* alpha, int32_t alpha_per_request,
                                const int32_t* ctx_len, const int32_t* cap, int32_t B,
                                int32_t k_max, int32_t policy, tsv_latency_model target,
                                tsv_latency_model draft, double pld_cost_ms,
                                int64_t kv_free_slots, int32_t* k_out, double* goodput_out,
                                int32_t* k_per_request, void* stream);

/* Batched ArgMaxGoodput for sweeps (BASELINE config 5): n_inst independent
 * batches; instance n owns requests [inst_offsets[n], inst_offsets[n+1]) of the
 * concatenated ctx_len / cap arrays and the global alpha[n].  Outputs k_out[n],
 * goodput_out[n*(k_max+1) + k] (nullable), k_per_request (nullable, same layout
 * as ctx_len).  Bit-identical to one tsv_goodput_choose_k per instance; one CTA
 * per instance. */
TSV_API tsv_status tsv_goodput_choose_k_batched(const double* alpha, const int32_t* ctx_len, const int32_t* cap,
                                                const int32_t* inst_offsets, int32_t n_inst, int32_t k_max,
                                                int32_t policy, tsv_latency_model target, tsv_latency_model draft,
                                                double pld_cost_ms, int64_t kv_free_slots, int32_t* k_out,
                                                double* goodput_out, int32_t* k_per_request, void* stream);

/* --------------------------------------------------------------------------
 * Fused Propose + GetVerificationLen for the PLD method (Listing 1 lines 15-16 +
 * 22-23): tsv_propose_lookup followed by tsv_goodput_choose_k
 * with policy TSV_POLICY_PLD, cap = the proposal lengths just found and
 * k_max = k_fixed, in ONE kernel: every CTA adds its request's terms of the
 * batch sums (exact int64 atomics) after its lookup, and the CTA that arrives
 * last evaluates the goodput of each k and writes k*, the goodput values and k_i.
 * Outputs are identical to the two separate calls.
 *   counter  device scratch of TSV_LOOKUP_CHOOSE_SCRATCH bytes (8-byte aligned),
 *            zero-filled once after allocation (tsv_workspace_clear); every call
 *            leaves it zero.  One per stream.  NULL: TSV_ERR_WORKSPACE.
 *   device_status as tsv_propose_lookup.
 * ------------------------------------------------------------------------ */
#define TSV_LOOKUP_CHOOSE_SCRATCH 512
TSV_API tsv_status tsv_propose_lookup_choose_k(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                                       int32_t n_min, int32_t n_max, int32_t k_fixed,
                                       int32_t* proposals, int32_t* proposal_len,
                                       const double* alpha, int32_t alpha_per_request,
                                       const int32_t* ctx_len, tsv_latency_model target,
                                       double pld_cost_ms, int64_t kv_free_slots, int32_t* k_out,
                                       double* goodput_out, int32_t* k_per_request,
                                       uint32_t* counter, int32_t* device_status, void* stream);
/* With flags: TSV_LOOKUP_INPUTS_READY as for tsv_propose_lookup_ex, the inputs
 * being ctx, ctx_offsets, ctx_len and alpha and the outputs proposals,
 * proposal_len, k_out, goodput_out and k_per_request: the search, the batch
 * sums and the last CTA's ArgMaxGoodput all run before the grid-dependency
 * wait.
 *   alpha_ready  nullable device word: before reading alpha the kernel waits
 *                (acquire, bounded: TSV_DEVSTATUS_WAIT_TIMEOUT) until it is 1.
 *                With the previous step's tsv_verify_accept_update_ex (which
 *                resets the word in its first kernel and sets it once alpha is
 *                written) and TSV_VERIFY_EARLY_TRIGGER, this lookup + choose-k
 *                runs in the previous race's tail and still reads that step's
 *                alpha.  NULL: alpha must qualify as an input (written two or
 *                more kernels back). */
TSV_API tsv_status tsv_propose_lookup_choose_k_ex(const int32_t* ctx, const int32_t* ctx_offsets, int32_t B,
                                          int32_t n_min, int32_t n_max, int32_t k_fixed,
                                          int32_t* proposals, int32_t* proposal_len,
                                          const double* alpha, int32_t alpha_per_request,
                                          const int32_t* ctx_len, tsv_latency_model target,
                                          double pld_cost_ms, int64_t kv_free_slots, int32_t* k_out,
                                          double* goodput_out, int32_t* k_per_request,
                                          uint32_t* counter, int32_t* device_status,
                                          const uint32_t* alpha_ready, int32_t flags, void* stream);

/* --------------------------------------------------------------------------
 * Acceptance-rate update: UpdateGlobalAcceptance (Listing 1 line 19,
 * PAPER.md:219) with the moving average of PAPER.md:131-132:
 *   r = sum_i m_i / sum_i tested_i,  alpha' = fma(decay, alpha - r, r)   (R17)
 * tested_i = m_i + [m_i < k_i] (TSV_EST_TESTED, R18) or k_i (TSV_EST_PROPOSED);
 * k_i from row_offsets as in tsv_verify_accept; requests with m_i < 0 are
 * skipped; nothing tested -> alpha unchanged.  per_request != 0: alpha is
 * [B] and alpha_i is updated from request i alone (R19).
 * ------------------------------------------------------------------------ */
#define TSV_EST_TESTED 0
#define TSV_EST_PROPOSED 1

TSV_API tsv_status tsv_update_acceptance(double* alpha, int32_t per_request, const int32_t* num_accepted,
                                 const int32_t* row_offsets, int32_t B, double decay,
                                 int32_t estimator, void* stream);

/* Fused Accept + UpdateGlobalAcceptance (Listing 1 lines 18-19): tsv_verify_accept
 * followed by tsv_update_acceptance(alpha, per_request, a->num_accepted,
 * a->row_offsets, a->B, decay, estimator), with the update run beside the race by the
 * race grid's last warp when it has no work item (else by one extra CTA of the race
 * kernel) -- the accepted counts are final after the acceptance scan, so it needs no
 * handshake.  Outputs identical to the two
 * separate calls; same workspace as tsv_verify_accept. */
TSV_API tsv_status tsv_verify_accept_update(const tsv_verify_args* a, double* alpha, int32_t per_request,
                                    double decay, int32_t estimator, void* stream);
/* ... with alpha_ready (nullable device word): the call's first kernel sets it to 0
 * (after its grid-dependency wait) and the update sets it to 1 (release) once
 * alpha is written -- the signal a following kernel that may start before this
 * call completes (TSV_VERIFY_EARLY_TRIGGER) waits on before reading alpha, e.g.
 * tsv_propose_lookup_choose_k_ex(..., alpha_ready, TSV_LOOKUP_INPUTS_READY).
 * Initialise the word to 1 (alpha valid) before the first call. */
TSV_API tsv_status tsv_verify_accept_update_ex(const tsv_verify_args* a, double* alpha, int32_t per_request,
                                       double decay, int32_t estimator, uint32_t* alpha_ready, void* stream);

/* --------------------------------------------------------------------------
 * Request-sharded step over NVLink peer memory (the exchange fused into
 * its producing kernels, no NCCL launch): every rank holds a disjoint set of the batch's
 * requests (global request ids) and one tsv_p2p handle (tsv_p2p_alloc/open/init below).
 *  tsv_goodput_choose_k_p2p: ONE kernel -- this rank's exact int64 ArgMaxGoodput sums
 *    (tsv_goodput_partial), summed over the ranks through peer memory, then Listing 2 on
 *    the global sums (tsv_goodput_finalize): k*, goodput and k_i = min(k*, cap_i) for the
 *    local requests, bit-identical to one device holding the whole batch.  B may be 0
 *    (the rank still takes part).  Arguments as tsv_goodput_choose_k.
 *  tsv_update_acceptance_p2p: UpdateGlobalAcceptance with (sum m, sum t) summed over the
 *    ranks before the EWMA (every rank applies the same update); per_request != 0 updates
 *    the local alphas with no exchange.
 *  tsv_verify_accept_update_p2p: tsv_verify_accept_update whose update warp / CTA (beside
 *    the race) performs that exchange -- the global alpha costs no extra launch.
 * All ranks must make the same sequence of exchange calls (tsv_goodput_choose_k_p2p,
 * tsv_update_acceptance_p2p, tsv_verify_accept_update_p2p, tsv_allreduce_i64_p2p share
 * one epoch).  device_status (nullable) gets TSV_DEVSTATUS_P2P_TIMEOUT.
 * ------------------------------------------------------------------------ */
TSV_API tsv_status tsv_goodput_choose_k_p2p(const double* alpha, int32_t alpha_per_request, const int32_t* ctx_len,
                                            const int32_t* cap, int32_t B, int32_t k_max, int32_t policy,
                                            tsv_latency_model target, tsv_latency_model draft, double pld_cost_ms,
                                            int64_t kv_free_slots, int32_t* k_out, double* goodput_out,
                                            int32_t* k_per_request, tsv_p2p* p, int32_t* device_status, void* stream);
TSV_API tsv_status tsv_update_acceptance_p2p(double* alpha, int32_t per_request, const int32_t* num_accepted,
                                             const int32_t* row_offsets, int32_t B, double decay, int32_t estimator,
                                             tsv_p2p* p, int32_t* device_status, void* stream);
TSV_API tsv_status tsv_verify_accept_update_p2p(const tsv_verify_args* a, double* alpha, int32_t per_request,
                                                double decay, int32_t estimator, tsv_p2p* p, void* stream);

/* Latency-model fit (reading R25; "fits a linear regression
 * model"): ordinary least squares of ms[i] on (ctx_tokens[i],
 * batched_tokens[i], 1) over n >= 3 HOST samples; while a coefficient is negative,
 * clamp every negative one to 0 and refit the remaining ones.  Writes the model
 * and (nullable) R^2 of the final fit.  Host-only (no device work).  Errors:
 * TSV_ERR_INVALID_ARG for n < 3 (TooFewSamples) or collinear regressors
 * (DegenerateDesign). */
TSV_API tsv_status tsv_fit_latency_model(const double* ctx_tokens, const double* batched_tokens, const double* ms,
                                         int32_t n, tsv_latency_model* out, double* r2_out);

/* --------------------------------------------------------------------------
 * Closed-loop harness (reading R26): a synthetic target
 * and the context append close the decode loop on the device -- lookup ->
 * choose-k -> tsv_sim_target -> verify (+ alpha update) -> tsv_context_append --
 * so the controller's adaptation can be replayed for many steps
 * as one CUDA graph without model weights.  All pointers are device pointers.
 * tsv_sim_target: request i verifies k_req[i] drafts proposals[i*K + j]; writes
 *   row_offsets [B+1] (exclusive scan of k_req + 1), drafts (packed at
 *   row_offsets[i] - i), row_info [rows_cap] scratch, and p_out rows [rows_cap, ld]:
 *   draft row j puts *alpha_true on x_j and (1 - *alpha_true)/(V - 1) elsewhere,
 *   the bonus row is uniform 1/V; columns >= V are 0.  rows_cap >= B (K + 1).
 *   With q = NULL in the verify, each draft is kept with probability *alpha_true.
 * tsv_context_append: windows of L tokens (request i at [iL, (i+1)L)); appends the
 *   num_accepted[i] + 1 emitted tokens (out_tokens [B, k_max+1]) and drops the
 *   oldest, writing ctx_out (must not alias ctx_in); ctx_len[i] += num_accepted[i]+1
 *   (unchanged for flagged requests, num_accepted < 0).
 * ------------------------------------------------------------------------ */
TSV_API tsv_status tsv_sim_target(const int32_t* proposals, int32_t K, const int32_t* k_req, int32_t B,
                                  const float* alpha_true, int32_t V, int64_t ld, int32_t rows_cap, float* p_out,
                                  int32_t* row_offsets, int32_t* drafts, int32_t* row_info, void* stream);
TSV_API tsv_status tsv_context_append(const int32_t* ctx_in, int32_t L, int32_t B, const int32_t* out_tokens,
                                      const int32_t* num_accepted, int32_t k_max, int32_t* ctx_out, int32_t* ctx_len,
                                      void* stream);

/* --------------------------------------------------------------------------
 * Communicator for the multi-GPU modes (NCCL over NVLink 5 / NVSwitch,
 * resolved at run time from the process's libnccl.so.2).
 * tsv_comm_get_unique_id: rank 0 only; the 128 bytes are broadcast by the
 * caller (torch.distributed).  tsv_verify_accept_sharded: lazy two rounds
 * (flags -> ncclAllReduce sum -> race -> ncclAllReduce max -> emit), or with
 * flags & TSV_VERIFY_SHARD_DENSE one round (partial -> ncclAllGather of
 * tsv_shard_tuple rows -> combine), all on `stream`; workspace >=
 * tsv_verify_sharded_workspace_size.
 * tsv_allreduce_i64: in-place sum of `count` int64 on `stream` (request-
 * sharded global sums for the alpha update and choose-k).
 * ------------------------------------------------------------------------ */
typedef struct tsv_comm tsv_comm;

TSV_API tsv_status tsv_comm_get_unique_id(void* unique_id_out /* 128 bytes */);
TSV_API tsv_status tsv_comm_init(tsv_comm** out, const void* unique_id, int32_t rank, int32_t world);
TSV_API tsv_status tsv_comm_destroy(tsv_comm* comm);
TSV_API tsv_status tsv_verify_sharded_workspace_size(const tsv_verify_args* a, int32_t world, size_t* bytes);
TSV_API tsv_status tsv_verify_accept_sharded(const tsv_verify_args* a, tsv_comm* comm, void* stream);
TSV_API tsv_status tsv_allreduce_i64(int64_t* data, size_t count, tsv_comm* comm, void* stream);

/* --------------------------------------------------------------------------
 * Request-sharded goodput and alpha update (one exchange step).
 * Every batch-level quantity ArgMaxGoodput and
 * UpdateGlobalAcceptance need is an exact integer sum over
 * requests, so each rank reduces its own requests and the element-wise sum
 * over ranks equals the unsharded batch's sums: k*, goodput and alpha are bit-
 * identical to one device holding the whole batch, for any partition.
 *
 * tsv_goodput_partial: sums[TSV_GP_SUMS(k_max)] (int64, device) of this rank's
 *   B >= 0 requests: [0..K] L(k) = sum_i rint(2^32 l(alpha_i, min(k, cap_i))),
 *   [K+1..2K+1] N(k) = sum_i min(k, cap_i), then sum ctx_len, sum ctx_len over
 *   cap_i > 0, #{cap_i > 0}, B.  Arguments as tsv_goodput_choose_k.
 * tsv_goodput_finalize: ArgMaxGoodput on (summed) sums -> k_out, goodput_out
 *   [k_max+1] (nullable); k_per_request[i] = min(k*, cap[i]) for this rank's
 *   B_local requests (both nullable).
 * tsv_goodput_choose_k_sharded: partial -> ncclAllReduce(sum) -> finalize on
 *   `stream`; sums_ws: int64[TSV_GP_SUMS(k_max)] device scratch.
 * tsv_update_partial: sums[2] = (sum_i m_i, sum_i t_i) over valid requests
 *   (t_i per `estimator`); tsv_update_finalize: alpha' = fma(d, alpha - r, r),
 *   r = sum_m / sum_t, unchanged when sum_t = 0 (global alpha only).
 * tsv_update_acceptance_sharded: partial -> ncclAllReduce(sum) -> finalize;
 *   sums_ws: int64[2] device scratch.
 * ------------------------------------------------------------------------ */
#define TSV_GP_SUMS(k_max) (2 * ((k_max) + 1) + 4)
TSV_API tsv_status tsv_goodput_partial(const double* alpha, int32_t alpha_per_request, const int32_t* ctx_len,
                                       const int32_t* cap, int32_t B, int32_t k_max, int64_t* sums, void* stream);
TSV_API tsv_status tsv_goodput_finalize(const int64_t* sums, int32_t k_max, int32_t policy, tsv_latency_model target,
                                        tsv_latency_model draft, double pld_cost_ms, int64_t kv_free_slots,
                                        const int32_t* cap, int32_t B_local, int32_t* k_out, double* goodput_out,
                                        int32_t* k_per_request, void* stream);
TSV_API tsv_status tsv_goodput_choose_k_sharded(const double* alpha, int32_t alpha_per_request,
                                                const int32_t* ctx_len, const int32_t* cap, int32_t B, int32_t k_max,
                                                int32_t policy, tsv_latency_model target, tsv_latency_model draft,
                                                double pld_cost_ms, int64_t kv_free_slots, int32_t* k_out,
                                                double* goodput_out, int32_t* k_per_request, int64_t* sums_ws,
                                                tsv_comm* comm, void* stream);
TSV_API tsv_status tsv_update_partial(const int32_t* num_accepted, const int32_t* row_offsets, int32_t B,
                                      int32_t estimator, int64_t* sums, void* stream);
TSV_API tsv_status tsv_update_finalize(double* alpha, const int64_t* sums, double decay, void* stream);
TSV_API tsv_status tsv_update_acceptance_sharded(double* alpha, const int32_t* num_accepted,
                                                 const int32_t* row_offsets, int32_t B, double decay,
                                                 int32_t estimator, int64_t* sums_ws, tsv_comm* comm,
                                                 void* stream);

/* --------------------------------------------------------------------------
 * Diagnostics (used by the GPU tests; not on the hot path).
 * tsv_debug_race_E: out[t] = E(u) of the race uniform u = (2(m_begin+t)+1) 2^-24
 *   exactly as the race kernels evaluate it (series near u = 1, double log
 *   elsewhere), for t < n, m_begin + n <= 2^23.  out: fp32 [n] device.
 * tsv_debug_philox: out[4t..4t+3] = Philox4x32-10(ctr[4t..4t+3], key[0..1]) on the
 *   device; race_variant != 0 uses the row-specialised evaluation of the race
 *   kernels (philox_race).  ctr: uint32 [4n], key: uint32 [2], out: uint32 [4n].
 * tsv_debug_race_row: one warp races the weights w[V] with the given Philox words
 *   (one per element, instead of generated ones) through the race kernels' logic
 *   (prune != 0: the prune test and deferred exact evaluation; 0: every element
 *   exact) and writes the packed key (bits(score) << 32 | ~v, 0 = no positive
 *   weight) to *key_out (device uint64).
 * ------------------------------------------------------------------------ */
TSV_API tsv_status tsv_debug_race_row(const float* w, const uint32_t* words, int32_t V, int32_t prune,
                                      uint64_t* key_out, void* stream);
TSV_API tsv_status tsv_debug_race_E(uint32_t m_begin, uint32_t n, float* out, void* stream);
TSV_API tsv_status tsv_debug_philox(const uint32_t* ctr, const uint32_t* key, uint32_t n, uint32_t* out,
                                    int32_t race_variant, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TSV_H */
