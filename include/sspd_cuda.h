/*
 * sspd_cuda.h -- the drop-in boundary: a C ABI over the B200 (sm_100a)
 * implementation of the sliding super point detector hot path
 * (arXiv 1803.11036; reference /root/reference/proj).
 *
 * Plain pointers and sizes only; no C++ or torch types.  The C++ API in
 * include/sspd/ (the reference's public headers, re-implemented in
 * paper_1803_11036_b200/csrc/host/) sits on top of these entry points, and so
 * do the Python bindings (paper_1803_11036_b200/_cabi.py) and any other
 * FFI.  Each entry point names the reference interface it
 * replaces (file:line, relative to /root/reference/proj).
 *
 * Representation.  The grid holds one u32 "slice stamp" per recorder instead
 * of the reference's u16 distance.  A per-grid counter `now` starts at 65535
 * and advance_slot increments it; stamp 0 means never seen.  The reference's
 * distance of a recorder is min(now - stamp, 0xFFFF), bit-exactly, so
 * advance_slot is O(1), union-min merge is element-wise max of stamps and
 * paper-max merge is element-wise min.  Touches are first recorded in a
 * per-slot bitmap (1 bit per recorder) and folded into the stamps by an
 * ordered pass before anything reads the grid; see DESIGN.md.
 *
 * Errors.  Every call returns an sspd_status; sspd_last_error() gives the
 * message of the last failure on the calling thread, worded like the
 * reference's exception text so the C++ shim can rethrow the same exception
 * types with the same what().
 *
 * Threading.  Calls on one grid are serialised by a per-grid mutex, so
 * concurrent scan callers (the reference's SCAN phase contract,
 * rsea.hpp:49-51) remain legal.  Work is queued on the grid's CUDA stream;
 * calls that return host data synchronise that stream.
 */
#ifndef SSPD_CUDA_H
#define SSPD_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SSPD_OK = 0,
  SSPD_INVALID_ARGUMENT = 1,  /* std::invalid_argument in the reference */
  SSPD_OUT_OF_RANGE = 2,      /* std::out_of_range */
  SSPD_CANDIDATE_OVERFLOW = 3,/* sspd::CandidateOverflow (rsea.hpp:38-43) */
  SSPD_CUDA_ERROR = 4,        /* device failure -> std::runtime_error */
  SSPD_NO_DEVICE = 5          /* no usable sm_100 device: fail loudly */
} sspd_status;

typedef enum { SSPD_UNION_MIN = 0, SSPD_PAPER_MAX = 1 } sspd_merge_policy; /* snapshot.hpp:11-14 */

typedef struct sspd_grid sspd_grid;

/* One reported host: the reference's Detection (rsea.hpp:25-28) plus the
 * integer in-window count the estimate was computed from. */
typedef struct {
  uint32_t cip;
  uint32_t r_k;
  double estimate;
} sspd_detection;

/* ---- library ---- */
int sspd_abi_version(void);
const char* sspd_last_error(void);
/* Number of visible devices this library can run on (sm_100). */
sspd_status sspd_device_count(int* n);
/* Their CUDA ordinals, ascending (up to cap of them; *n = how many there
 * are).  On a mixed box these are not 0..n-1. */
sspd_status sspd_device_ordinals(int* out, int cap, int* n);

/* ---- device memory, for hosts that wire routers together in one process
 * (the C++ run_detection over several GPUs, csrc/host/routers.cpp) ---- */
sspd_status sspd_device_alloc(int device, uint64_t bytes, void** ptr);
sspd_status sspd_device_free(int device, void* ptr);
/* Device blocks of >= 1 MiB freed by grids (and sspd_device_free) are kept
 * for reuse -- a grid's create + destroy would otherwise cost tens of ms of
 * cudaMalloc/cudaFree -- up to $SSPD_CACHE_BYTES per device (default 16 GiB).
 * This frees them (device < 0: every device); *released (may be NULL) gets
 * the byte count.  Allocation failures flush the cache by themselves. */
sspd_status sspd_release_cached(int device, uint64_t* released);
/* Pairwise peer access among the listed devices (NVLink loads/stores). */
sspd_status sspd_enable_peer_access(int n_devices, const int* devices);
/* Synchronous copy on the grid's stream: host -> device (to_device != 0) or
 * device -> host. */
sspd_status sspd_grid_copy(sspd_grid* g, void* dst, const void* src, uint64_t bytes, int to_device);

/* ---- grid lifetime: Rsea::Rsea (rsea.hpp:54; rsea.cpp:18-27) ---- */
/* Validates like validate_config(cfg, eta, 1, 1.0) (hashing.cpp:63-87) and
 * fails with "Rsea: <first diagnostic>".  All recorders start never-seen. */
sspd_status sspd_grid_create(int device, uint32_t q, uint32_t r, uint32_t delta,
                             uint64_t seed, uint32_t eta, sspd_grid** out);
/* B200 extension (BASELINE config C4's stamp-width axis): a grid whose
 * recorders hold `width`-bit stamps (8 or 16; 32 = sspd_grid_create plus
 * sspd_track_window(k_max)).  Narrow grids are exact for in-window counts
 * with k <= k_max and everything derived from them -- active_counts,
 * hot_sets, finalize, reconstruct -- and keep the window ring on; k_max must
 * be below 2^width - 1.  Entry points that need full distances or stamps
 * (get/put_distances, clone, merge, equal, commit, the exchange hooks) fail
 * with SSPD_INVALID_ARGUMENT on them. */
sspd_status sspd_grid_create_narrow(int device, uint32_t q, uint32_t r, uint32_t delta,
                                    uint64_t seed, uint32_t eta, uint32_t width,
                                    uint32_t k_max, sspd_grid** out);
/* A sharded router's PARTIAL grid: only the cells router `rank` of `world`
 * owns (cell c belongs to c * world / (r * 2^q)) get stamps on `device`,
 * so N routers hold an N-times larger table between them.  k_max > 0 also
 * tracks the window ring.  Scans need sspd_set_shard(_relay) with the same
 * world and rank first; distances are readable for the owned recorders only
 * (sspd_grid_owned); calls that need every cell (clone, merge, equal,
 * reconstruct, finalize, hot_sets, active_counts, the other exchange hooks)
 * fail with SSPD_INVALID_ARGUMENT. */
sspd_status sspd_grid_create_sharded(int device, uint32_t q, uint32_t r, uint32_t delta, uint64_t seed,
                                     uint32_t eta, uint32_t k_max, uint32_t world, uint32_t rank,
                                     sspd_grid** out);
/* Recorders [rec_lo, rec_hi) held by this grid (everything unless partial). */
sspd_status sspd_grid_owned(const sspd_grid* g, uint64_t* rec_lo, uint64_t* rec_hi);
/* Stamp width (8, 16, 32) and tracked window (0 = none). */
sspd_status sspd_grid_stamp_width(const sspd_grid* g, uint32_t* width, uint32_t* k_max);
/* Copy constructor (Rsea is copyable: snapshot.cpp:127, pipeline.cpp:39):
 * device-to-device copy onto `device` (-1 = the source's device). */
sspd_status sspd_grid_clone(const sspd_grid* src, int device, sspd_grid** out);
sspd_status sspd_grid_destroy(sspd_grid* g);
/* Geometry and state: recorder_count (rsea.hpp:59), device, now. */
sspd_status sspd_grid_info(const sspd_grid* g, uint64_t* recorders, int* device,
                           uint32_t* now);
/* Queue the grid's work on an external cudaStream_t (NULL = the grid's own). */
sspd_status sspd_grid_set_stream(sspd_grid* g, void* cuda_stream);
/* The cudaStream_t the grid's work is queued on (its own or the one set). */
sspd_status sspd_grid_stream(const sspd_grid* g, void** cuda_stream);
sspd_status sspd_grid_synchronize(sspd_grid* g);

/* ---- SCAN phase ---- */
/* Rsea::scan_batch / Rsea::update (rsea.hpp:71-75; rsea.cpp:29-53).  `pairs`
 * holds n (cip, oip) u32 pairs interleaved (the IpPair layout, rsea.hpp:14-17).
 * pairs_on_device != 0: device pointer on the grid's device, consumed in place;
 * otherwise a host pointer, copied in chunks on a copy stream that overlaps
 * the scan.  Pinned input is copied by DMA as it lies (the call returns once
 * the copies are done); pageable input (>= 4096 pairs) is packed into pinned
 * staging by host worker threads first.  Order- and batch-invariant like
 * the reference. */
sspd_status sspd_scan(sspd_grid* g, const uint32_t* pairs, uint64_t n, int pairs_on_device);
/* The same over n (ts, cip, oip) trace records (workload.hpp TraceRecord,
 * 12 bytes each; ts is ignored -- the caller picks a slot's records).  Device
 * and pinned records are turned into pairs on the device; pageable ones are
 * packed as pairs while being staged (8 of every 12 bytes cross PCIe).  A
 * time-sorted trace is scanned slot run by slot run, with no copy of it. */
sspd_status sspd_scan_records(sspd_grid* g, const uint32_t* records, uint64_t n, int on_device);

/* ---- QUIESCENT phase ---- */
/* Rsea::advance_slot (rsea.cpp:55-63): O(1), `slots` times. */
sspd_status sspd_advance(sspd_grid* g, uint32_t slots);

/* Rsea::cells() as distances (rsea.hpp:61-68): recorders [offset, offset+count)
 * in (row, column, bucket) order, as the reference's u16 values. */
sspd_status sspd_get_distances(sspd_grid* g, uint16_t* host_out, uint64_t offset,
                               uint64_t count);
/* Writes through a mutable cells() span (import_snapshot, snapshot.cpp:95-111). */
sspd_status sspd_put_distances(sspd_grid* g, const uint16_t* host_in, uint64_t offset,
                               uint64_t count);

/* rec::active_count over every estimator (estimator.hpp:26-31): R_k per cell,
 * r*2^q values in (row, column) order. */
sspd_status sspd_active_counts(sspd_grid* g, uint32_t k, uint32_t* host_out);

/* Rsea::hot_sets (rsea.cpp:65-84) with the integer cutoff
 * hot_cutoff(eta, theta) computed by the caller (estimator.cpp:32-36).
 * cols_out: capacity r*2^q, rows concatenated, columns ascending;
 * row_counts: r entries. */
sspd_status sspd_hot_sets(sspd_grid* g, uint32_t k, uint64_t cutoff, uint32_t* cols_out,
                          uint32_t* row_counts);

/* Rsea::finalize_candidate (rsea.cpp:86-108) over n tuples of r columns
 * (host memory).  accepted[i] = 1 when tuple i is accepted, with cip/r_k
 * filled.  The estimate is estimate_cardinality(eta, r_k) on the host. */
sspd_status sspd_finalize(sspd_grid* g, const uint32_t* tuples, uint64_t n, uint32_t k,
                          uint64_t cutoff, uint8_t* accepted, uint32_t* cips,
                          uint32_t* r_ks);

/* Rsea::reconstruct_leveled (rsea.cpp:168-255): hot cells, level-2 triples,
 * levels 3..r-1, finalize, dedup by cip (larger estimate kept) sorted by cip.
 * Fails with SSPD_CANDIDATE_OVERFLOW and *ovf_level / *ovf_count set exactly
 * as CandidateOverflow(level, count, cap) would be.  Writes at most out_cap
 * detections; *n_out is the full count.  The same cip set as
 * reconstruct_recursive (rsea.cpp:126-166), which has no cap (pass
 * cap = UINT64_MAX).  Supports r <= 64 (as does sspd_finalize). */
sspd_status sspd_reconstruct(sspd_grid* g, uint32_t k, uint64_t cutoff, uint64_t cap,
                             sspd_detection* out, uint64_t out_cap, uint64_t* n_out,
                             uint32_t* ovf_level, uint64_t* ovf_count);

/* B200 extension: sspd_reconstruct split in two so a stream of slots
 * pipelines.  _async queues the whole reconstruction (hot sets, joins,
 * finalize, the read-back of counts and survivors) on the grid's stream and
 * returns at once; _collect waits for it and returns what sspd_reconstruct
 * would have (reports, or SSPD_CANDIDATE_OVERFLOW with level and count).
 * Scans and advances may be queued in between: the stream orders them after
 * the reconstruction, which sees the grid as of the _async call.  One
 * reconstruction may be queued per grid; sspd_reconstruct, sspd_finalize and
 * the shard calls refuse while it is.  Candidate buffers are sized for `cap`
 * up front (cap <= 2^26). */
sspd_status sspd_reconstruct_async(sspd_grid* g, uint32_t k, uint64_t cutoff, uint64_t cap);
sspd_status sspd_reconstruct_collect(sspd_grid* g, sspd_detection* out, uint64_t out_cap,
                                     uint64_t* n_out, uint32_t* ovf_level, uint64_t* ovf_count);

/* merge_rseas (snapshot.hpp:54; snapshot.cpp:117-142): element-wise combine
 * of n grids into `out` (which may alias grids[0] for an in-place merge).
 * Grids must share (seed, q, r, delta, eta) -- else SSPD_INVALID_ARGUMENT with
 * the reference's message -- and are brought to a common `now`.  Grids on other
 * devices are read directly over NVLink (peer access). */
sspd_status sspd_merge(const sspd_grid* const* grids, uint64_t n, int policy,
                       sspd_grid* out);

/* Rsea::operator== (rsea.hpp:100-102): same distances everywhere. */
sspd_status sspd_equal(sspd_grid* a, sspd_grid* b, int* equal);

/* ---- window tracking (B200-native extension) ---- */
/* Maintain per-cell in-window counts incrementally for windows up to k_max
 * slots, so hot_sets / reconstruct at k <= k_max skip the full-grid count
 * pass.  0 disables.  Results are identical either way. */
sspd_status sspd_track_window(sspd_grid* g, uint32_t k_max);

/* ---- sharded routers (B200 extension; paper_1803_11036_b200/dist.py SHARD) ----
 * Router `rank` of `world` owns the cells c with c * world / (r * 2^q) == rank
 * (a contiguous slice) and keeps exact stamps only there.  Its own scans stamp
 * owned recorders and push each pair new to the router to the owners of the
 * pair's other cells: P2P stores into dev_inbox_ptrs[owner] (a device array of
 * `world` peer-mapped inbox bases, each world * region_cap (cip, oip) pairs;
 * region `rank` of an inbox is this router's).  Per slot, after the scans:
 *   sspd_shard_sent      device u64[world]: pairs pushed to each owner (the
 *                        caller all-gathers them; a count past region_cap is
 *                        an error the caller must raise);
 *   sspd_shard_receive   scan the pairs peers pushed here (owned cells only);
 *   sspd_shard_hot       this router's hot bits (device u32 words): OR them
 *                        across routers in place;
 *   sspd_shard_select    joins and address checks on the merged hot sets, then
 *                        per-survivor bucket masks (device u32): AND them
 *                        across routers in place;
 *   sspd_shard_finish    R_k = popcount of the merged masks; reports as
 *                        sspd_reconstruct.
 * The reports equal sspd_reconstruct on the union-min merge of the routers'
 * grids.  world = 0 turns sharding off. */
sspd_status sspd_set_shard(sspd_grid* g, void* dev_inbox_ptrs, uint32_t world, uint32_t rank,
                           uint64_t region_cap);
/* Relayed sharding (two hops): the scan pushes each new pair only to its
 * pair owner (a hash of the pair mod world) through inbox table A; the pair
 * owner runs sspd_shard_relay over what it received (all sources, itself
 * included), which dedups the routers' union for its share, stamps its own
 * cells and pushes each pair once to the other cell owners through table B;
 * cell owners then sspd_shard_receive what arrived (no second dedup needed).
 * sspd_shard_sent's counters: [0, 32) hop 1, [32, 64) hop 2. */
sspd_status sspd_set_shard_relay(sspd_grid* g, void* dev_inbox_a, void* dev_inbox_b, uint32_t world,
                                 uint32_t rank, uint64_t region_cap);
sspd_status sspd_shard_relay(sspd_grid* g, const uint32_t* dev_pairs, uint64_t n);
/* sspd_shard_relay over n_regions inbox regions in ONE launch: region i holds
 * counts[i] (host array) pairs at dev_base + 2 * i * region_stride words.
 * (One launch pads each warp's list blocks once instead of once per region.) */
sspd_status sspd_shard_relay_regions(sspd_grid* g, const uint32_t* dev_base, uint64_t region_stride,
                                     const uint64_t* counts, uint32_t n_regions);
/* The same with the counts read by the kernel from DEVICE memory (no host
 * round trip in the slot): region i holds dev_counts[i * count_stride] pairs,
 * e.g. this router's column of the all-gathered `sent` counters.  A count
 * past region_stride is clamped and flagged (sspd_shard_overflow). */
sspd_status sspd_shard_relay_regions_dev(sspd_grid* g, const uint32_t* dev_base, uint64_t region_stride,
                                         const uint64_t* dev_counts, uint64_t count_stride, uint32_t n_regions);
sspd_status sspd_shard_sent(sspd_grid* g, uint64_t** dev_counts);
sspd_status sspd_shard_receive(sspd_grid* g, const uint32_t* dev_pairs, uint64_t n);
/* sspd_shard_receive over n_regions inbox regions in one launch, counts in
 * device memory as above; region skip_region (this router's own) is empty. */
sspd_status sspd_shard_receive_regions_dev(sspd_grid* g, const uint32_t* dev_base, uint64_t region_stride,
                                           const uint64_t* dev_counts, uint64_t count_stride, uint32_t n_regions,
                                           uint32_t skip_region);
/* 1 if a device-counted region ran past its stride since the last call. */
sspd_status sspd_shard_overflow(sspd_grid* g, int* overflowed);
/* dst[w] = OR (op 0) or AND (op 1) over srcs[0..n_src)[w], w < words, in one
 * kernel on `device` (stream NULL = the legacy default stream).  srcs is a
 * host array of device pointers -- peers' buffers over NVLink (peer access or
 * symmetric memory) -- so routers merge hot bits and survivor masks without a
 * host round trip.  dst may not alias a source another device still reads. */
sspd_status sspd_reduce_words(int device, const uint32_t* const* srcs, uint32_t n_src, uint64_t words, int op,
                              uint32_t* dst, void* cuda_stream);
sspd_status sspd_shard_hot(sspd_grid* g, uint32_t k, uint64_t cutoff, uint32_t** dev_hot_words,
                           uint64_t* n_words);
sspd_status sspd_shard_select(sspd_grid* g, uint32_t k, uint64_t cutoff, uint64_t cap, uint64_t* n_surv,
                              uint32_t** dev_masks, uint64_t* mask_words, uint32_t* ovf_level,
                              uint64_t* ovf_count);
sspd_status sspd_shard_finish(sspd_grid* g, uint64_t cutoff, sspd_detection* out, uint64_t out_cap,
                              uint64_t* n_out);

/* ---- raw device views, for torch.distributed / NCCL plumbing ---- */
/* Device pointer to the u32 stamp array (recorders words) after folding any
 * pending touches.  Stamps are < 2^31, so an int32 view reduces identically. */
sspd_status sspd_grid_stamps(sspd_grid* g, uint32_t** dev_stamps, uint64_t* words);
/* Device pointer to this slot's touched bitmap (ceil(recorders/32) words)
 * without folding it, for an OR-merge across routers; after the caller has
 * OR-reduced it in place, sspd_commit folds it into the stamps. */
sspd_status sspd_grid_touched(sspd_grid* g, uint32_t** dev_bits, uint64_t* words);
sspd_status sspd_commit(sspd_grid* g);
/* Union-min exchange between routers.  mode 1: record each slot's touched
 * bitmap (OR-merge it, then sspd_commit).  mode 2: list each slot's distinct
 * (cip, oip) pairs (scans then always use the pair set); routers all-gather
 * the lists and scan each other's.  0: off. */
sspd_status sspd_set_exchange(sspd_grid* g, int mode);
/* Fused exchange (with mode 2): while scanning, also store each new pair into
 * every peer router's inbox over NVLink.  dev_peer_ptrs: device array of
 * `world` pointers (peer-mapped symmetric memory, e.g. torch
 * _SymmetricMemory.buffer_ptrs_dev), each the base of `world` regions of
 * `region_cap` (cip, oip) pairs; router `rank` writes region `rank` of every
 * other router's inbox at the position its pair has in the local list.
 * Positions >= region_cap are not pushed (the caller falls back to the list).
 * world <= 1 disables. */
sspd_status sspd_set_push(sspd_grid* g, void* dev_peer_ptrs, uint32_t world, uint32_t rank,
                          uint64_t region_cap);
/* This slot's new pairs (exchange mode 2): device pointer to `count`
 * interleaved (cip, oip) pairs, valid until the next advance.  Every pair new
 * to the grid this slot appears at least once; the list is grown in blocks
 * reserved per warp, whose unused tails hold copies of listed pairs (a
 * repeated pair changes nothing where it is applied). */
sspd_status sspd_grid_new_pairs(sspd_grid* g, uint32_t** dev_pairs, uint64_t* count);
/* Scan strategy: mode 0 = deferred bitmap, 1 = direct stamping, 2 = direct
 * behind a per-slot set of seen pairs, 3 = as 2 after partitioning large
 * device batches by pair-set region, -1 = auto (2 when the touched bitmap
 * would exceed 48 MiB, else 1);
 * filter 0/1 = L1 duplicate probe, -1 = keep.  Results are identical in
 * every mode, and modes may be mixed within a slot.  Narrow-stamp grids run
 * mode 0 as 1 and mode 3 as 2. */
sspd_status sspd_scan_mode(sspd_grid* g, int mode, int filter);
/* Keys found new to their slot by the pipelined dedup scan (the C2 path),
 * summed since the grid was created: the set's inserts plus probes that hit
 * the probe limit.  A key is (cip, bucket(oip)) on the key-set scan (eta <=
 * 2^16) and (cip, oip) otherwise.  Diagnostic (bench.py's per-launch fresh
 * keys; the key set's growth). */
sspd_status sspd_grid_fresh_pairs(sspd_grid* g, uint64_t* count);

/* The pipelined scan's per-slot key set (kernels.cuh scan_cset_kernel), for
 * tests and diagnostics: its device pointer (u32 entries, NULL before the
 * first key-set scan) and log2 of its entry count, after the grid's queued
 * work.  Valid until the next scan or advance. */
sspd_status sspd_grid_keyset(sspd_grid* g, uint32_t** dev_entries, uint32_t* log2_entries);
/* The CHECKED build (lib/libsspd_cuda_checked.so, -DSSPD_CHECKED): bounds
 * checks on every data-dependent stamp / code / window-ring index and the
 * ring's no-underflow invariant (kernels.cuh "CHECKED BUILD").  Waits for the
 * device, returns the first failing kernels.cuh line and the failure count,
 * optionally resetting both.  The product library returns
 * SSPD_INVALID_ARGUMENT. */
sspd_status sspd_checked_status(int device, uint32_t* first_line, uint64_t* failures, int reset);

/* ---- synthetic traces (shape of synth_trace,
 * workload.cpp:215-300), bit-identical on host and device ---- */
/* Parameters: see paper_1803_11036_b200/csrc/synth.h (sspd_synth_params). */
typedef struct {
  uint64_t seed;
  uint32_t hosts;
  uint32_t pool;
  uint32_t n_super;
  uint32_t super_fanout;
  uint64_t pairs_per_slot;
  uint32_t shard;
  uint32_t n_shards;
} sspd_synth_params_t;
/* Integer Zipf CDF over `hosts` ranks (hosts+0 entries, last = 2^63). */
sspd_status sspd_synth_zipf_cdf(uint32_t hosts, double exponent, uint64_t* cdf_out);
/* n pairs of slot `slot` starting at local index j0, into host memory
 * (all host cores) or device memory (cdf must then be a device pointer). */
sspd_status sspd_synth_host(const sspd_synth_params_t* p, const uint64_t* cdf, uint64_t slot,
                            uint64_t j0, uint64_t n, uint32_t* pairs_out);
sspd_status sspd_synth_device(int device, const sspd_synth_params_t* p, const uint64_t* dev_cdf,
                              uint64_t slot, uint64_t j0, uint64_t n, uint32_t* dev_pairs_out,
                              void* cuda_stream);
/* Distinct super point cips injected by the generator (ground truth for
 * the injected set). */
uint32_t sspd_synth_super_cip(const sspd_synth_params_t* p, uint32_t i);

/* Exact ground truth on the device: the number of distinct
 * oips of every cip over the union of n_segments device arrays of (cip, oip)
 * pairs (one sliding window's slots) -- what exact_counts reports for that
 * window (workload.cpp:180-213) -- for cips with count >= min_count, sorted
 * by cip.  distinct_hint sizes the tables (0 = total pairs); a full table
 * fails with SSPD_OUT_OF_RANGE rather than dropping anything. */
sspd_status sspd_exact_counts(int device, const uint32_t* const* dev_segments, const uint64_t* seg_pairs,
                              uint32_t n_segments, uint64_t distinct_hint, uint32_t min_count,
                              uint32_t* cips, uint32_t* counts, uint64_t out_cap, uint64_t* n_out,
                              void* cuda_stream);

/* Per-kernel timing of the last call on this grid (CUDA events on the grid's
 * stream), for bench.py's roofline: name -> milliseconds, launches. */
sspd_status sspd_profile_enable(sspd_grid* g, int on);
sspd_status sspd_profile_read(sspd_grid* g, const char* kernel, double* total_ms,
                              uint64_t* launches, uint64_t* units);
sspd_status sspd_profile_reset(sspd_grid* g);
/* Host<->device bytes this grid's calls have copied (e2e accounting). */
sspd_status sspd_grid_io_bytes(sspd_grid* g, uint64_t* h2d, uint64_t* d2h, int reset);
/* Total kernels this library has launched (all grids, since load). */
uint64_t sspd_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SSPD_CUDA_H */
