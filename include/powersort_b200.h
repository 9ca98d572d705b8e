/*
 * powersort_b200.h -- C ABI of the B200-native Multiway Powersort hot path.
 *
 * Drop-in boundary for the reference's sort entry point
 *   stable_sort_with(lst, config) -> SortStats
 *     (/root/reference/pkg/src/powersort/policy.py:201-262)
 * and its helpers node_power / run_stack_capacity (power.py:37-74) and
 * merge_cost_for_profile (policy.py:270-304).  Plain pointers and sizes only;
 * device pointers are CUDA global memory on the current device, `stream` is a
 * cudaStream_t (NULL = legacy default stream).
 *
 * Every entry point returns a ps_status; ps_last_error() gives a message.
 * The library has no CPU fallback: without a usable CUDA device every sort
 * call fails with PS_ECUDA.
 */
#ifndef POWERSORT_B200_H
#define POWERSORT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (the Python shim maps them to exceptions). */
typedef enum {
    PS_OK = 0,
    PS_EINVAL = 1,      /* ValueError: bad k / variant / min_run_len / bounds  */
    PS_ECUDA = 2,       /* RuntimeError: CUDA error or no device               */
    PS_ENOMEM = 3,      /* MemoryError: workspace too small / allocation       */
    PS_EINVARIANT = 4,  /* AssertionError: policy invariant (policy.py:114,139) */
    PS_EOVERFLOW = 5    /* OverflowError: run stack bound (policy.py:117-120)  */
} ps_status;

/* Key types.  Records are (key, int32 value); keys compare with IEEE `<=`
 * for floats (-0.0 == +0.0; NaN unsupported, as in the reference). */
typedef enum { PS_INT32 = 0, PS_INT64 = 1, PS_FLOAT32 = 2, PS_FLOAT64 = 3 } ps_dtype;

/* Merge-kernel families, policy.py:49-69 (VARIANTS).  The merge tree depends
 * only on (k, min_run_len, strict_merge_down); the variant selects the
 * counter formulas of merges.py:99-104, 141, 195-201, 270-275, 330-334, 395-399. */
typedef enum {
    PS_VARIANT_2WAY = 0,
    PS_VARIANT_2WAY_COPY_SMALLER = 1,
    PS_VARIANT_2WAY_NOSENTINEL = 2,
    PS_VARIANT_4WAY = 3,
    PS_VARIANT_4WAY_NOSENTINEL = 4
} ps_variant;

/* What happens to the int32 `values` array passed to ps_sort. */
typedef enum {
    PS_VALUES_PERMUTE = 0, /* values[] is a payload permuted alongside the keys      */
    PS_VALUES_ARGSORT = 1  /* values[] is output only: receives the source indices   */
} ps_values_mode;

/* SortConfig, policy.py:72-91 (key/on_merge live in the Python shim). */
typedef struct {
    int32_t k;                 /* 2 or 4 */
    int32_t variant;           /* ps_variant, must match k */
    int64_t min_run_len;       /* >= 1 (MIN_RUN_LEN = 24, policy.py:34-36) */
    int32_t strict_merge_down; /* policy.py:146-175 */
    int32_t values_mode;       /* ps_values_mode */
    int32_t count_comparisons; /* 1: exact comparisons / moves (CountingOrder, statskit.py:49-72) */
    int32_t flags;             /* PS_FLAG_* bits; 0 = the reference's synchronous contract */
} ps_config;

/* ps_config.flags.  Without PS_FLAG_ASYNC, ps_sort returns after the merges
 * have run and reports their device invariant flags (chunk bounds, grid
 * barriers) as PS_EINVARIANT, like the reference's assertions.  With it,
 * ps_sort returns once the merges are queued on `stream` (stats are already
 * final host values) and ps_check() reports the merge-phase flags later. */
enum { PS_FLAG_ASYNC = 1 };

/* SortStats, statskit.py:75-98 (scalar fields).  comparisons / moves are
 * data-dependent counters of the reference's sequential kernels; they are
 * computed when ps_config.count_comparisons is set (then *_valid is 1).  An
 * asynchronous sort (PS_FLAG_ASYNC) leaves them on the device: *_valid is 2
 * and ps_result_counters() returns them once the stream has finished. */
typedef struct {
    int64_t comparisons;
    int64_t merge_cost;
    int64_t buffer_cost;
    int64_t moves;
    int64_t max_stack_height;
    int64_t runs_detected;
    int64_t merges2;
    int64_t merges3;
    int64_t merges4;
    int64_t scan_reads;
    int64_t scan_writes;
    int32_t comparisons_valid;
    int32_t moves_valid;
} ps_stats;

/* Bytes of device workspace ps_sort needs for n keys of `dtype` under cfg.
 * Returns 0 on invalid arguments. */
size_t ps_workspace_size(int64_t n, int32_t dtype, const ps_config* cfg);

/* stable_sort_with(lst, config) on a device array: sorts keys[0..n) in place,
 * stably, permuting values[0..n) alongside (or writing the source indices,
 * PS_VALUES_ARGSORT).  Replaces policy.py:201-262 (with the run detection of
 * runs.py:23-82, the powers of power.py:47-74, the stack policy of
 * policy.py:94-175 and the merge kernels of merges.py:75-500).
 * `workspace` is device memory of >= ps_workspace_size() bytes; it also holds
 * the run profile and merge tree afterwards (see ps_result_*).
 * keys, values and workspace must be 16-byte aligned.
 * Returns after the merges have run and their device invariants were checked
 * (or, with PS_FLAG_ASYNC, once they are queued on `stream`; then ps_check()
 * synchronizes and reports merge-phase device invariants).  Concurrent sorts
 * on different streams need separate workspaces. */
int ps_sort(int32_t dtype, void* keys, int32_t* values, int64_t n, const ps_config* cfg, void* workspace,
            size_t workspace_bytes, ps_stats* stats, void* stream);

/* Synchronizes `stream` and returns PS_EINVARIANT if the last ps_sort on
 * `workspace` raised a device invariant flag during its merges. */
int ps_check(void* workspace, void* stream);

/* Number of runs r and merge nodes of the last ps_sort / ps_tree_from_profile
 * that used `workspace`. */
/* comparisons / moves of the last asynchronous counting sort on `workspace`
 * (ps_stats.*_valid == 2): synchronizes `stream`, checks the device invariant
 * flags, and returns them (-1 where the sort could not count exactly). */
int ps_result_counters(void* workspace, void* stream, int64_t* comparisons, int64_t* moves);

int ps_result_counts(const void* workspace, int64_t* runs, int64_t* merges);

/* Copy the run profile of the last sort to host arrays of length >= runs:
 * SortStats.run_lengths / natural_run_lengths (policy.py:241-248).
 * Either pointer may be NULL. */
int ps_result_runs(const void* workspace, int64_t* run_lengths, int64_t* natural_run_lengths, int64_t cap);

/* Copy the executed merge tree to host rows of 7 int64 in the reference's
 * on_merge order (policy.py:237-239): width, b0..b4 (b_width = end, rest -1),
 * output length. */
int ps_result_trace(const void* workspace, int64_t* rows, int64_t cap);

/* merge_cost_for_profile (policy.py:270-304) on the device tree builder:
 * builds the merge tree of a run-length profile (host array of r lengths).
 * Results are read with ps_result_counts / ps_result_trace. */
size_t ps_profile_workspace_size(int64_t r, int64_t n);
int ps_tree_from_profile(const int64_t* lengths, int64_t r, int32_t k, int32_t strict_merge_down,
                         void* workspace, size_t workspace_bytes, int64_t* merge_cost, int64_t* max_stack_height,
                         void* stream);

/* node_power (power.py:47-55): least p >= 1 with floor(A k^p / 2n) <
 * floor(B k^p / 2n), A = b1+e1, B = b2+e2; exact.  k in {2,3,4} (any k >= 2
 * when any_k != 0, as _node_power_any).  Returns p >= 1, or -PS_EINVAL. */
int ps_node_power(int32_t k, int64_t n, int64_t b1, int64_t e1, int64_t b2, int64_t e2, int32_t any_k);

/* run_stack_capacity (power.py:37-44): (k-1) * (ceil(log_k n) + 1). */
int64_t ps_run_stack_capacity(int64_t k, int64_t n);

/* Multi-GPU cross-shard merge.  Every rank g of G sorted its
 * contiguous shard (ps_sort with the shard's own n, payload = global index);
 * this call produces the rank's slab of the globally sorted sequence, global
 * ranks [out_begin, out_end) (normally [g*N/G, (g+1)*N/G)), in one pass that
 * reads the G shards directly (peer pointers over NVLink P2P; no NCCL, no
 * gathered copy).  shard_keys[i]/shard_vals[i] are device pointers valid on
 * the current device (local or peer-mapped), shard_n[i] their lengths; shard
 * i holds global indices [sum_{j<i} shard_n[j], ...).  shard_samples[i] is
 * shard i's sample array (ps_shard_samples) or NULL (the samples are then
 * read from the keys with a stride); shard_samples itself may be NULL.
 * out_keys/out_vals receive the slab.  Stable: ties ordered by shard then
 * position.  Stream-ordered; returns after one final synchronisation that
 * reads the device error flags.  No reference counterpart: the reference is
 * single-threaded; the merge is merges.py:204-275's stable
 * k-way merge with k = G <= 8. */
size_t ps_shard_merge_workspace_size(int32_t nshards, int64_t slab_n);
int ps_shard_merge(int32_t dtype, int32_t nshards, const void* const* shard_keys, const int32_t* const* shard_vals,
                   const void* const* shard_samples, const int64_t* shard_n, int64_t out_begin, int64_t out_end,
                   void* out_keys, int32_t* out_vals, void* workspace, size_t workspace_bytes, void* stream);

/* Peer shards for ps_shard_merge (plumbing for the multi-GPU mode only; no
 * reference counterpart).  ps_ipc_export writes the 64-byte cudaIpcMemHandle_t
 * of the allocation holding device pointer `ptr` and ptr's byte offset in it.
 * ps_ipc_open opens another process's handle in `device`'s context with lazy
 * peer access enabled, so kernels on `device` load from it over NVLink
 * (*base = the allocation's base; add the exporter's offset).  ps_ipc_close
 * unmaps it. */
int ps_ipc_export(int32_t device, const void* ptr, void* handle, int64_t* offset);
int ps_ipc_open(int32_t device, const void* handle, void** base);
int ps_ipc_close(int32_t device, void* base);

/* Sample array of a sorted shard for ps_shard_merge: samples[i] = keys[i *
 * stride], stride = 128 bytes of keys (32 four-byte or 16 eight-byte keys);
 * ps_shard_sample_count gives the array length, ceil(n / stride). */
int64_t ps_shard_sample_count(int32_t dtype, int64_t n);
int ps_shard_samples(int32_t dtype, const void* keys, int64_t n, void* samples, void* stream);

/* Payloads of any width: dst row i = src row perm[i], rows
 * of row_bytes bytes, for the permutation a PS_VALUES_ARGSORT sort returned.
 * src and dst must not overlap.  Stream-ordered; device pointers. */
int ps_gather_rows(const void* src, const int32_t* perm, void* dst, int64_t n, int64_t row_bytes, void* stream);

/* Phase timing of ps_sort (CUDA events on the sort's stream).  Enabled per
 * host thread; ps_profile_read returns the entries of the last profiled sort.
 * kind: 0 run detection, 1 merge tree, 2 leaf formation, 3 cut partition,
 * 4 merge launch.  bytes = algorithmic HBM bytes of the entry: merges read
 * and write every record once (2 * sum(node sizes) * record bytes). */
typedef struct {
    int32_t kind;
    int32_t stage;   /* merge stage index (power levels high..low, then merge_down) */
    int64_t nodes;
    int64_t chunks;
    int64_t bytes;
    float ms;
    float pad;
} ps_prof_entry;

int ps_profile_enable(int32_t on);
int ps_profile_read(ps_prof_entry* out, int32_t cap, int32_t* count);

/* Number of kernels this library has launched in this process. */
int64_t ps_launch_count(void);

/* Message for the last non-OK status on this thread. */
const char* ps_last_error(void);

/* Library version string. */
const char* ps_version(void);

#ifdef __cplusplus
}
#endif

#endif /* POWERSORT_B200_H */
