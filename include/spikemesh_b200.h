/*
 * spikemesh-b200 C ABI -- the drop-in boundary of the sm_100a construction
 * and propagation path of arXiv 2512.09502 (reference package `spikemesh`
 * 0.1.0, cited as sm/<file>:<line> = /root/reference/pkg/src/spikemesh/...).
 *
 * Conventions
 *   - every function is `extern "C"`, takes plain pointers and sizes, and
 *     returns an int status: 0 ok, -1 ValueError, -2 ConsistencyError,
 *     -3 CUDA error, -4 ProtocolError, -5 DelayRangeError (the reference's
 *     exception classes, sm/core.py:39-52); smx_last_error() has the text;
 *   - pointers are DEVICE pointers unless named *_host; `stream` is a
 *     cudaStream_t (pass 0 for the legacy default stream);
 *   - stream keys are the two Philox key words (k0, k1) of
 *     RngStream(seed, stream_id) (sm/core.py:119-126): k0 | k1 << 64 =
 *     int.from_bytes(blake2b(canonical_bytes((seed, stream_id)), 16), "little");
 *   - u32 cursors count 32-bit draws consumed from the start of a stream
 *     (numpy's next_uint32 buffering), word cursors count 64-bit words.
 * Library: paper_2512_09502_b200/_build/libspikemesh_b200.so
 */
#ifndef SPIKEMESH_B200_H
#define SPIKEMESH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- plumbing ------------------------------------------------------------ */
int smx_last_error(char* buf, size_t cap);
const char* smx_version(void);
int smx_stream_sync(void* stream);
/* host wait policy for synchronisations, before context creation
 * (cudaDeviceScheduleSpin = 1, Yield = 2, BlockingSync = 4) */
int smx_set_sync_policy(int flags);
/* Device-side chaining of draws on one keyed stream (sm/construction.py:
 * 424-431: fixed_total's targets continue after its positions; 157-176: a
 * syn stream's delays continue after its normal weights).  The next draw
 * entry point called on this thread starts at *u0_dev (u32 cursor, device;
 * null: its u0 argument) and writes its end cursor to *cursor_dev (device;
 * null: as usual), with no host synchronisation.  Taken once. */
int smx_draw_chain(const uint64_t* u0_dev, uint64_t* cursor_dev);
/* SMs pass A (smx_fused_gen) leaves empty for work on other streams -- the
 * replays and small kernels of the calls that follow (0..16, default 8).
 * Process-wide; a single-rank construction uses 0. */
int smx_set_pass_a_free_sms(int n);
/* A non-blocking stream (no implicit synchronisation with the legacy
 * default stream) at the given priority; the engine runs the fused path's
 * pass A and the preparation side work on such streams. */
int smx_stream_create(int priority, void** out);
/* keep the default stream-ordered pool's memory mapped (no trim at sync);
 * no reuse of blocks through inserted cross-stream waits */
int smx_pool_setup(int device);
/* device error word of asynchronous paths: read + clear (synchronises stream) */
int smx_check_device_errors(void* stream);
int* smx_device_error_word(void);
/* kernels launched by the library so far (process-wide counter) */
uint64_t smx_launch_count(void);

/* --- keyed streams (numpy 2.3.5 Generator(Philox) semantics) -------------
 * Replaces RngStream (sm/core.py:110-148) draws made by the construction
 * path: integers at sm/construction.py:169,402,406,426,430,527,679 and
 * sm/models.py:175-178; normal at :160,:362; poisson at sm/dynamics.py:233. */
int smx_philox_words(uint64_t k0, uint64_t k1, uint64_t w0, uint64_t n, uint64_t* out, void* stream);
/* Generator.integers(lo, lo+ex, size=n) (int64) from u32 cursor; ex in [1, 2^32]. */
int smx_integers(uint64_t k0, uint64_t k1, uint64_t u32_cursor, int64_t lo, uint64_t ex, uint64_t n,
                 int64_t* out, uint64_t* cursor_out_host, void* stream);
/* v[i] = RngStream(seed, (..., gids[i])).normal(mu, sd), canonical bytes of the
 * stream id = prefix + decimal(gid) + suffix (sm/construction.py:361-365). */
int smx_init_v(const uint8_t* prefix_host, uint32_t plen, const uint8_t* suffix_host, uint32_t slen,
               const int64_t* gids, uint64_t n, double mu, double sd, double* v_out, void* stream);
int smx_stream_keys(const uint8_t* prefix_host, uint32_t plen, const uint8_t* suffix_host, uint32_t slen,
                    const int64_t* ids, uint64_t n, uint64_t* keys_out, void* stream);
/* Generator.poisson(lam < 10, size=n) from the word cursor *cursor_in;
 * writes the cursor after the last sample to *cursor_out (no host sync).
 * Workspace: smx_poisson_workspace(smx_poisson_chunks_for(n, lam)) bytes. */
uint64_t smx_poisson_workspace(int n_chunks);
int smx_poisson_chunks_for(uint64_t n, double lam);
int smx_poisson_counts(uint64_t k0, uint64_t k1, const uint64_t* cursor_in, double enlam, uint64_t n,
                       int n_chunks, void* workspace, uint8_t* counts, uint64_t* cursor_out, int* err,
                       void* stream);
/* lam >= 10: numpy random_poisson_ptrs (two words per trial), same chain
 * machinery and contract; counts above 255 set the error flag. */
int smx_poisson_counts_ptrs(uint64_t k0, uint64_t k1, const uint64_t* cursor_in, double lam, uint64_t n,
                            int n_chunks, void* ws, uint8_t* counts, uint64_t* cursor_out, int* err, void* stream);

/* --- construction ---------------------------------------------------------
 * Replaces sm/construction.py:391-703 (rule realization, flag/extract,
 * image maps, remap) and ConnectionStore.append_batch (sm/core.py:257-293).
 * Pending records are (u32 key, u32 payload): key = source node, or
 * 0x80000000 | lut index for remote-call records whose image ids are
 * assigned after generation; payload = target row | syn class << 24. */
int smx_pay_table(const int64_t* targets, uint64_t n, const int32_t* node2row, uint64_t n_nodes, uint32_t cls,
                  uint32_t* pay_tab, void* stream);
int smx_key_table(const int64_t* sources, uint64_t n, uint32_t tmp_base, int tmp, uint32_t* key_tab, void* stream);
int smx_dist_tables(const int32_t* src_rank, const int64_t* src_node, uint64_t total, const uint32_t* vbase,
                    int tgt_rank, uint32_t lut_base, uint32_t* key_tab, uint32_t* gv_tab, void* stream);
/* One Generator.integers(0, ex, size=n) draw routed into pending records:
 * key_mode 0 none / 1 key_tab[value] / 2 key_tab[j / kdiv] /
 *          3 piecewise-affine key = value + delta[s] for start[s] <= value,
 *            key_tab then being a HOST array {n (<= 8), start[n], delta[n]};
 * pay_mode 0 none / 1 pay_tab[value] / 2 pay_tab[j / kdiv];
 * used_bits (optional, used_bits_words words) marks bit
 * used_tab ? used_tab[value] : value for every emitted draw, or with
 * mark_from_key the bit of the record key: (key & ~TMP) - tmp_base for
 * temporary keys, local_bit for direct ones.  cursor_out_host may be NULL:
 * then nothing is read back (no host synchronisation) and a draw window short
 * of accepted draws (12-sigma margin) is reported by smx_check_device_errors. */
int smx_gen_draw(uint64_t k0, uint64_t k1, uint64_t u32_cursor, uint64_t ex, uint64_t n, int key_mode,
                 int pay_mode, const uint32_t* key_tab, const uint32_t* pay_tab, uint32_t kdiv, uint32_t* keys,
                 uint32_t* vals, uint32_t* used_bits, const uint32_t* used_tab, uint32_t used_bits_words,
                 int mark_from_key, uint32_t tmp_base, uint32_t local_bit, uint64_t* cursor_out_host,
                 void* stream);
/* counts[s] += number of keys in [lo[s], hi[s]) for m <= 16 disjoint ranges;
 * ranges_host = {m, lo[m], hi[m]}.  Records per source rank of one
 * distributed call, for the modeled-byte accounting (sm/construction.py:689-703,
 * 597-617). */
int smx_count_ranges(const uint32_t* keys, uint64_t n, const uint32_t* ranges_host, unsigned long long* counts,
                     void* stream);
/* allow_multapses=False: rows x k values of numpy Generator.choice(n, k,
 * replace=False), one row per target, back to back from u32 cursor u32_cursor
 * (sm/core.py:140-141, sm/construction.py:403-404, 680-683). */
int smx_choice_rows(uint64_t k0, uint64_t k1, uint64_t u32_cursor, uint64_t n, uint64_t k, uint64_t rows,
                    uint32_t* values, uint64_t* cursor_out_host, void* stream);
/* records from drawn positions: keys[j] = key_tab ? key_tab[v] : v, vals[j] =
 * pay_tab[j / kdiv]; optional used-value bits (mark_tab ? mark_tab[v] : v). */
int smx_records_from_values(const uint32_t* values, uint64_t n, const uint32_t* key_tab, const uint32_t* pay_tab,
                            uint32_t kdiv, uint32_t* keys, uint32_t* vals, uint32_t* bits,
                            const uint32_t* mark_tab, void* stream);
/* one_to_one / assigned (mode 0), all_to_all (mode 1): sm/construction.py:415-419 */
int smx_gen_pairs(int mode, uint64_t n, uint64_t n_src, const uint32_t* key_tab, const uint32_t* pay_tab,
                  uint32_t* keys, uint32_t* vals, void* stream);
/* allow_autapses=False redraw loop of local fixed_indegree / fixed_total
 * calls (sm/construction.py:524-529), continuing the call's stream at u0. */
int smx_autapse_fix(uint64_t k0, uint64_t k1, uint64_t u0, uint64_t n_src, const uint32_t* key_tab, uint32_t* keys,
                    const uint32_t* rows, uint64_t n, const int32_t* node2row, uint64_t n_nodes,
                    uint64_t* cursor_out_host, void* stream);
/* used_flags + extract_used (sm/construction.py:454-470) as a value bitmap */
int smx_mark_values(const uint32_t* pos_bits, const int64_t* sources, uint64_t n, uint32_t* vbits, void* stream);
/* lookup_or_create_images + RemoteSourceMap.insert (sm/construction.py:473-486,
 * 227-236); segs_host: array of {u64 word0, u64 nwords, u32* present, i32* img_of}. */
int smx_assign_images(const uint32_t* vbits, uint64_t nwords, const void* segs_host, int n_segs, int64_t m0,
                      int64_t* n_new_host, void* stream);
/* remap_connection_sources (sm/construction.py:489-495) via the key LUT */
int smx_gather_lut(const int64_t* sources, uint64_t n, const int32_t* img_of, uint32_t* lut, void* stream);
/* mirror_merge / roster update (sm/construction.py:295-306, 633-636) */
int smx_bits_or(uint32_t* dst, const uint32_t* src, uint64_t nwords, void* stream);
/* dst |= src[0] | ... | src[n-1] (srcs_host: host array of device pointers) */
int smx_bits_or_many(uint32_t* dst, const uint32_t* const* srcs_host, int n_srcs, uint64_t nwords, void* stream);
int smx_bits_prefix(const uint32_t* bits, uint64_t nwords, int64_t* excl, void* stream);
int smx_bits_compact(const uint32_t* bits, uint64_t nwords, const int64_t* excl, int64_t* out,
                     const int32_t* img_of, int64_t* img_out, void* stream);
int smx_fill_wide_const(double* w, uint32_t* meta, uint64_t n, double wv, uint32_t mv, void* stream);
/* _realize_syn random specs (sm/construction.py:157-176): normal weights
 * (numpy Generator.normal from word cursor *cursor_in; workspace as for the
 * Poisson counts with smx_normal_chunks_for(n) chunks) and uniform_int delays
 * (integers from u32 cursor u0) written as meta = delay | port << 24. */
int smx_normal_chunks_for(uint64_t n);
int smx_normal_fill(uint64_t k0, uint64_t k1, const uint64_t* cursor_in, double loc, double scale, uint64_t n,
                    int n_chunks, void* workspace, double* values, uint64_t* cursor_out, int* err, void* stream);
int smx_delay_fill(uint64_t k0, uint64_t k1, uint64_t u0, uint32_t lo, uint64_t ex, uint64_t n, uint32_t port,
                   uint32_t* meta, uint64_t* cursor_out_host, void* stream);
int smx_promote_wide(const uint32_t* vals, uint64_t n, const double* cls_w, const uint32_t* cls_meta,
                     uint32_t* rows, double* w, uint32_t* meta, void* stream);

/* --- preparation (sm/construction.py:742-807, sm/core.py:299-324) ---------- */
/* Fused construction path (csrc/fused.cu).  The reference's
 * fixed-in-degree realisation (sm/construction.py:391-406, 640-703) and the
 * stable store sort (ConnectionStore.finalize, sm/core.py:299-324) as two
 * passes of an LSD radix sort whose first pass is the draw itself.
 * smx_fused_gen: one call's integers(0, ex, size=n_out) draws from the start
 * of stream (k0, k1), ranked by the low key digit and written as packed u32
 * records (key >> lo_bits) << pbits | (pay_tab[j / kdiv] & 0xffffff) | cls_field
 * (cls_field = the call's class index << its row bits) into the digit regions
 * (rstart / rcap / fill_in / fill_out: device arrays of 2^lo_bits entries;
 * pay_tab: smx_pay_table's row | class << 24 of each target).
 * key_mode 3: key_tab is a host array {n, start[n], delta[n]} of piecewise-
 * affine keys; key_mode 1: device table key_tab[value].  *total_out = accepted
 * draws of the raw window (< n_out: window short); *overflow set when a region
 * was too small (the caller rebuilds through smx_gen_draw + smx_sort_records). */
int smx_fused_gen(uint64_t k0, uint64_t k1, uint64_t ex, uint64_t n_out, int key_mode, const uint32_t* key_tab,
                  uint32_t kdiv, const uint32_t* pay_tab, uint32_t cls_field, int lo_bits, int pbits,
                  uint32_t* region, uint64_t n_slots,
                  const uint64_t* rstart, const uint64_t* rcap, const uint64_t* fill_in, uint64_t* fill_out,
                  uint64_t* total_out, int* overflow, void* stream);
/* smx_fused_sort: pass B over the regions (region digit * per_digit + call
 * at rptr[region], fill[region] records): stable scatter by the high digit
 * (hi_bits 8..11) writing out[] = row | cls_map[class index] in key order
 * and counts[key] (key = hi << lo_bits | digit; first_index via
 * smx_counts_to_offsets).  rcap_host: host copy of the capacities;
 * row_bits_host[call] (host, per_digit <= 512 entries): the call's payload
 * split, class index << row_bits | row (rows fixed at the call's time). */
int smx_fused_sort(const uint64_t* rptr, const uint64_t* fill, const uint64_t* rcap_host, int per_digit,
                   int lo_bits, int hi_bits, int pbits, const uint8_t* row_bits_host, const uint32_t* cls_map,
                   uint32_t* counts,
                   uint64_t n_keys, uint64_t n_records, uint32_t* out, int* err, void* stream);
/* ConnectionStore.finalize: stable sort of pending records by source. */
int smx_sort_records(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b, uint64_t n,
                     int key_bits, int index_values, const uint32_t* lut, uint32_t* counts, uint64_t n_keys,
                     int* out_in_b_host, void* stream);
/* first_index = exclusive scan of per-source counts (np.add.at + np.cumsum) */
int smx_counts_to_offsets(const uint32_t* counts, uint64_t n, int64_t* first_index, void* stream);
int smx_gather_wide(const uint32_t* idx, uint64_t n, const uint32_t* rows_in, const double* w_in,
                    const uint32_t* meta_in, uint32_t* rows, double* w, uint32_t* meta, void* stream);
/* out3 = {max delay, max port, min delay} of wide records */
int smx_max_meta(const uint32_t* meta, uint64_t n, uint32_t* out3, void* stream);
/* _build_point_routes / _build_group_routes (sm/construction.py:710-739);
 * tabs_host: array of {u32* bits, i64* excl, u64 nwords, i32 dest}. */
int smx_build_routes(const void* tabs_host, int nt, uint64_t n_nodes, uint32_t* cnt_scratch, int64_t* first,
                     int32_t* dest, uint32_t* pos, int64_t* n_entries_host, void* stream);

/* --- propagation (sm/engine.py:277-310) ----------------------------------- */
/* consume_inputs + kernels.lif_step (sm/dynamics.py:191-204,
 * kernels/_speedups.pyx:13-35) on real rows; ring is [L][P][n] fp64. */
int smx_lif_update(double* v, int32_t* ref, const double* decay, const double* v_rest, const double* v_reset,
                   const double* v_th, const int32_t* ref_steps, const double* i_e, uint32_t n, double* ring,
                   int n_ports, int L, const int64_t* now_dev, uint32_t* spike_bits, void* stream);
/* PoissonSource.emit_into (sm/dynamics.py:235-248) from a batch of
 * precomputed counts [S][n_t]; step taken from the device counter *now_dev. */
int smx_poisson_emit(const uint8_t* counts, int S, uint32_t n_t, const uint32_t* rows, double w, double* ring,
                     uint32_t n_rows, int n_ports, int L, int delay, int port, const int64_t* now_dev, void* stream);
/* flatnonzero + recorder + route_point_spikes / route_group_spikes
 * (sm/engine.py:89-128); p2p/grp: {i64* first, i32* dest, u32* pos, int n_dest,
 * u32* packets, u32* counts, u32 cap} (host structs). */
int smx_spikes(const uint32_t* spike_bits, uint32_t n_rows, const uint32_t* row2node, const int64_t* gid,
               int64_t* now_dev, uint32_t* src_nodes, uint32_t* src_steps, uint32_t* n_src, uint32_t src_cap,
               const int* record_dev, int64_t* rec, uint64_t* n_rec, uint64_t rec_cap, uint32_t* spike_count,
               int* overflow, const void* p2p_host, const void* grp_host, void* stream);
/* Spike exchange over NVLink peer memory (csrc/peer.cu), one process per
 * GPU: the data movement of LockstepTransport's rounds (sm/transport.py:
 * 92-168) without NCCL.  smx_peer_alloc / smx_peer_handle / smx_peer_open /
 * smx_peer_close / smx_peer_free: an IPC-exportable receive area and its
 * mapping in the senders.  smx_peer_exchange: per block, n_send PeerSend
 * descriptors (count, packets, receiver slot + flag per parity, capacity,
 * byte-count flag) and n_slot PeerSlot descriptors (local slot + flag per
 * parity, position lookup L / I, capacity): sends, then wait + unpack into
 * the delivery list (src_nodes, src_steps, *n_src).  *seq (device) is the
 * block sequence, *sent / *over the round's counters, *done a zeroed word. */
int smx_peer_alloc(uint64_t bytes, void** ptr);
int smx_peer_free(void* ptr);
int smx_peer_handle(void* ptr, void* handle_out);
int smx_peer_open(const void* handle, void** ptr);
int smx_peer_close(void* ptr);
int smx_peer_exchange(const void* sends_host, int n_send, const void* slots_host, int n_slot,
                      unsigned long long* seq, unsigned long long* sent, int* over, uint32_t* src_nodes,
                      uint32_t* src_steps, uint32_t* n_src, uint32_t src_cap, int* err, unsigned int* done,
                      uint32_t* zero0, uint32_t nzero0, uint32_t* zero1, uint32_t nzero1, void* stream);
/* deliver_point_packets / deliver_gather_packets (sm/engine.py:146-190).
 * *count (written by the sender) is clamped to max_count, the block's
 * capacity; a larger count sets *err = 5. */
int smx_unpack(const uint32_t* packets, const uint32_t* count, uint32_t max_count, const int64_t* table,
               uint64_t table_len, uint32_t* src_nodes, uint32_t* src_steps, uint32_t* n_src, uint32_t src_cap,
               int* err, void* stream);
/* kernels.deliver_spikes (kernels/_speedups.pyx:38-54) over a device list of
 * (source node, emission step); packed (cls_*) or wide (wide_w/wide_meta). */
int smx_deliver(const uint32_t* src_nodes, const uint32_t* src_steps, const uint32_t* n_src, uint32_t* wprefix,
                uint32_t* n_work, const int64_t* first, const uint32_t* payload, const double* cls_w,
                const uint32_t* cls_delay, const uint32_t* cls_port, const double* wide_w,
                const uint32_t* wide_meta, double* ring, uint32_t n_rows, int n_ports, int L, int grid,
                void* stream);

/* One complete local step (sm/engine.py:285-296) in three launches: fused
 * consume + LIF + Poisson emission + spike compaction + raster + packet
 * routing; local delivery; step-counter advance.  devs_host: array of
 * {u8* counts[S][n_t], i32* inv (row -> target index or -1), u32 n_t,
 * double w, int delay, int port} (Poisson devices with unique target rows); the step is *now_dev +
 * step_offset; ctr: 2 x u64 list counters indexed by step parity; owner:
 * work item -> list entry scratch. */
int smx_step(double* v, int32_t* ref, const double* decay, const double* v_rest, const double* v_reset,
             const double* v_th, const int32_t* ref_steps, const double* i_e, uint32_t n, double* ring, int n_ports,
             int L, int64_t* now_dev, int step_offset, const int* record_dev, int S, const void* devs_host, int n_dev,
             const uint32_t* row2node, const int64_t* gid, const int64_t* first, uint32_t* src_nodes,
             uint32_t* src_steps, uint32_t* wbase, uint32_t* owner, uint32_t owner_cap, unsigned long long* ctr,
             uint32_t src_cap, int64_t* rec, unsigned long long* n_rec, uint64_t rec_cap, int* err,
             const void* p2p_host, const void* grp_host, const uint32_t* payload, const double* cls_w,
             const uint32_t* cls_delay, const uint32_t* cls_port, const double* wide_w, const uint32_t* wide_meta,
             void* stream);

/* A block of n_steps local steps in two launches when every record delay
 * is >= n_steps (Poisson devices are applied by the target row's thread):
 * per-thread multi-step LIF with state in registers, then one
 * delivery of all the block's spikes.  Same arguments as smx_step plus
 * n_steps; ctr[0] is the block's list counter. */
int smx_block(double* v, int32_t* ref, const double* decay, const double* v_rest, const double* v_reset,
              const double* v_th, const int32_t* ref_steps, const double* i_e, uint32_t n, double* ring, int n_ports,
              int L, int64_t* now_dev, int step_offset, int n_steps, const int* record_dev, int S,
              const void* devs_host, int n_dev, const uint32_t* row2node, const int64_t* gid, const int64_t* first,
              uint32_t* src_nodes, uint32_t* src_steps, uint32_t* wbase, uint32_t* owner, uint32_t owner_cap,
              unsigned long long* ctr, uint32_t src_cap, int64_t* rec, unsigned long long* n_rec, uint64_t rec_cap,
              int* err, const void* p2p_host, const void* grp_host, const uint32_t* payload, const double* cls_w,
              const uint32_t* cls_delay, const uint32_t* cls_port, const double* wide_w, const uint32_t* wide_meta,
              void* stream);

/* --- reference-layout drop-ins for sm/kernels (kernels/__init__.py:25-26) ---
 * lif_step (_speedups.pyx:13-35): v f64[n], ref_count i64[n], real_mask u8[n],
 * inputs f64[n], decay/v_rest/v_reset/v_th f64[n], ref_steps i64[n],
 * spiked_out u8[n]. */
int smx_ref_lif_step(double* v, int64_t* ref_count, const uint8_t* real_mask, const double* inputs,
                     const double* decay, const double* v_rest, const double* v_reset, const double* v_th,
                     const int64_t* ref_steps, uint8_t* spiked_out, uint64_t n, void* stream);
/* deliver_spikes (_speedups.pyx:38-54): src_nodes/mults i64[k], first_index
 * i64[M+1], tgt/port/delay i64[S], weight f64[S], buffers f64[M][P][L]. */
int smx_ref_deliver_spikes(const int64_t* src_nodes, const int64_t* mults, uint64_t k, const int64_t* first_index,
                           const int64_t* tgt, const int64_t* port, const int64_t* delay, const double* weight,
                           double* buffers, int64_t n_ports, int64_t L, int64_t now, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPIKEMESH_B200_H */
