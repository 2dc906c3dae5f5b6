/*
 * crossover_sgd.h — C ABI of the B200-native Crossover-SGD gossip step.
 *
 * Method: Yeo et al., "Crossover-SGD: A gossip-based communication in distributed
 * deep learning for alleviating large mini-batch problem and enhancing
 * scalability", arXiv 2012.15198.  Citations are PAPER.md line numbers
 * (section / algorithm line) of /root/reference/PAPER.md; readings C-n are listed
 * in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Return 0 (CS_OK) on success, a negative CS_E* code on error; no exception
 *    ever crosses the ABI.  cs_last_error() gives a human-readable message for
 *    the calling thread's last error.
 *  - Device pointers are plain CUDA device addresses on the current device;
 *    host pointers are ordinary (or pinned) host memory.  The caller owns every
 *    buffer it passes; the library owns its topology tables, diagnostics
 *    scratch, staging buffers and peer-visible exchange region.
 *  - Device-side work is enqueued asynchronously on the bound stream.
 *    Device-detected conditions (non-finite gradient) surface as CS_EDIVERGED
 *    at the next cs_sync() / cs_get_diag().
 *  - One process-wide context (cs_init .. cs_finalize).  Not thread-safe.
 *  - There is no CPU fallback: every compute entry point runs CUDA kernels and
 *    fails with CS_ECUDA if no sm_100a device is usable.
 */
#ifndef CROSSOVER_SGD_H
#define CROSSOVER_SGD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------------- */
#define CS_OK                 0
#define CS_EINVAL_WORLD      -1   /* world < 2, world > CS_MAX_WORLD, or world % nprocs != 0 */
#define CS_EINVAL_GROUPS     -2   /* groups < 1 or groups does not divide world          */
#define CS_EINVAL_SEGMENTS   -3   /* k < 1, k > CS_MAX_SEGMENTS, or k > ceil(d/32)       */
#define CS_ELAYOUT           -4   /* misaligned pointer, ld % 4 != 0, ld < d, d < 1       */
#define CS_ETOPOLOGY         -5   /* Alg. 2 restart limit (10,000 attempts) exceeded      */
#define CS_EINVAL_TOPOLOGY   -6   /* injected topology row is not a derangement           */
#define CS_ENOTINIT          -7   /* cs_init has not been called                          */
#define CS_ENOTBOUND         -8   /* cs_bind has not been called                          */
#define CS_ECUDA             -9   /* CUDA runtime / launch failure (see cs_last_error)    */
#define CS_EDIVERGED        -10   /* a non-finite gradient was seen         */
#define CS_EINVAL           -11   /* other invalid argument (NULL pointer, step range)    */
#define CS_EUNSUPPORTED     -12   /* valid request this build does not implement          */
#define CS_ETIMEOUT         -13   /* a cross-GPU wait exceeded its bound                  */

#define CS_MAX_WORLD       1024   /* device Alg. 2 keeps a 1024-bit availability mask     */
#define CS_MAX_SEGMENTS    4096
#define CS_QUANTUM           32   /* segment bounds are multiples of 32 elements (C-2)    */
#define CS_MAX_LAYERS     65536   /* layer-table entries (cs_set_layers)                  */
#define CS_IPC_HANDLE_BYTES  64   /* sizeof(cudaIpcMemHandle_t)                           */

#define CS_TAG_FLAT 0             /* Philox domain tag of the flat topology               */
#define CS_TAG_HIER 1             /* Philox domain tag of the leader topology (C-13)      */

/* Topology kinds (cs_set_topology_kind). */
#define CS_TOPO_CROSSOVER   0   /* Alg. 2 load-balanced random topology per segment (default) */
#define CS_TOPO_EXPONENTIAL 1   /* SGP's directed exponential graph, the baseline */

/* Wire formats of exchanged segments (cs_set_wire). */
#define CS_WIRE_FP32 0   /* received segments in fp32 (default; the fp32 step of the paper)   */
#define CS_WIRE_BF16 1   /* received segments rounded to bf16; master state stays fp32 (C-20) */

/* ---- context -------------------------------------------------------------- */

/* Create the process-wide context.
 *   world      n = total number of workers across all processes (2..CS_MAX_WORLD).
 *   groups     G = number of hierarchical groups; must divide world.  Groups are
 *              contiguous blocks of world/G workers and the lowest rank of each
 *              block is its leader (§3.3; reading C-12).  G = world
 *              is the flat method; cs_gossip_step ignores G.
 *   k_segments k = number of segments the flat parameter vector is split into
 *              (reading C-2).
 *   seed       the "random seed which is shared by every process"
 *              — the Philox4x32-10 key of every topology draw (reading C-4).
 * Pure host call (no CUDA).  Re-initialising replaces any previous context.
 * Errors: CS_EINVAL_WORLD, CS_EINVAL_GROUPS, CS_EINVAL_SEGMENTS. */
int cs_init(int world, int groups, int k_segments, uint64_t seed);

/* Release every library-owned resource (device tables, peer mappings). */
void cs_finalize(void);

/* Message of the calling thread's most recent error ("" if none).  Owned by the
 * library; valid until the next cs_* call on this thread. */
const char* cs_last_error(void);

/* ABI version (major*10000 + minor*100 + patch). */
int cs_version(void);

/* Build id: the first 16 hex digits of the sha256 of the library's sources, this header and
 * the nvcc flags it was compiled from (static string; "unknown-build-id" if built by hand). */
const char* cs_build_id(void);

/* ---- pure host functions (callable before cs_bind, no GPU needed) ---------- */

/* Segment plan (reading C-2): bounds_out[s] = min(d, 32*floor(s*ceil(d/32)/k)),
 * bounds_out[k] = d.  bounds_out is caller-owned int64[k+1].
 * Errors: CS_ENOTINIT, CS_ELAYOUT (d < 1), CS_EINVAL_SEGMENTS (k > ceil(d/32)). */
int cs_segment_bounds(int64_t d, int64_t* bounds_out);

/* Topology of a flat step (§3.2 Alg. 2, readings C-1, C-4..C-7):
 * fills the caller-owned host int32 [k][world] with src_out[s*world + i] = the
 * worker that worker i RECEIVES segment s from at `step` (Alg.1 l.5
 * "receive_from = destinations[my rank]").  Every row is a
 * permutation without fixed points.  Pure function of (seed, step, world, k).
 * Requires 0 <= step < 2^32.  Errors: CS_ENOTINIT, CS_EINVAL, CS_ETOPOLOGY. */
int cs_topology(int64_t step, int32_t* src_out);

/* Leader topology of a hierarchical step (reading C-13): int32 [k][groups],
 * indices are dense leader indices 0..G-1, domain tag CS_TAG_HIER.
 * Errors as cs_topology; CS_EINVAL_GROUPS if groups < 2 (no leader gossip). */
int cs_topology_hier(int64_t step, int32_t* src_out);

/* ---- binding device state ------------------------------------------------- */

/* Register the caller's device state and this process's place in the job.
 *   momentum   fp32 device [n_loc][ld] heavy-ball buffer (reading C-9), updated
 *              in place by every step.  n_loc = world / nprocs local workers;
 *              local row r is global worker proc_rank*n_loc + r.
 *   d          parameters per worker (>= 1).   ld  row stride in elements
 *              (ld >= d, ld % 4 == 0, so rows are 16-byte aligned for 128-bit
 *              access).  Elements [d, ld) of a row are never written.
 *   proc_rank, nprocs   this process's index and the number of processes (one
 *              per GPU).  nprocs == 1: all workers co-resident on this GPU.
 *              nprocs > 1: call cs_ipc_export / cs_ipc_import next.
 *   stream     cudaStream_t to enqueue on (NULL = legacy default stream).
 * Buffers must be 16-byte aligned.  Allocates the library's device tables.
 * Errors: CS_ENOTINIT, CS_EINVAL_WORLD, CS_ELAYOUT, CS_EINVAL_SEGMENTS, CS_ECUDA. */
int cs_bind(float* momentum, int64_t d, int64_t ld, int proc_rank, int nprocs, void* stream);

/* Change the stream later steps are enqueued on. */
int cs_set_stream(void* stream);

/* Kernel path for later cs_bind calls (default CS_PATH_AUTO):
 *   CS_PATH_AUTO   nprocs > 1: CS_PATH_PEER; else CS_PATH_TMA when world <= 64 and
 *                  k*world <= 2048, otherwise CS_PATH_REG
 *   CS_PATH_REG    single-GPU column-owner kernel with register pipelining
 *   CS_PATH_TMA    single-GPU column-owner kernel with bulk-TMA row-tile staging
 *   CS_PATH_PEER   exchange-through-inbox kernel of the multi-GPU path; with
 *                  nprocs == 1 every receiver is local (single-GPU emulation of the
 *                  multi-GPU protocol, used by tests and profiling)
 * All paths compute bit-identical results.  Errors: CS_ENOTINIT, CS_EINVAL,
 * CS_EUNSUPPORTED (TMA requested for a topology it does not cover). */
#define CS_PATH_AUTO 0
#define CS_PATH_REG  1
#define CS_PATH_TMA  2
#define CS_PATH_PEER 3
int cs_set_path(int path);

/* Schedule of the multi-GPU flat step (applies now and to later cs_bind calls):
 *   CS_SCHED_INSTEP    (default) the merge a5 of a step completes inside that step's
 *                      enqueued work: when the stream reaches the end of cs_gossip_step,
 *                      params / psw hold x', w' ("parameter averaging is
 *                      processed after the gradient is applied"; Alg.1 l.12-17).  One worker
 *                      per GPU: one launch (k_push_merge: update, NVLink push and per-tile
 *                      landed-progress flags, in-kernel merge).  Several: walk + tail merge.
 *   CS_SCHED_DEFERRED  (opt-in) the merge of step t runs inside step t+1's kernel; params
 *                      hold y_t in between, so cs_flush / cs_sync must precede any read.
 *   CS_SCHED_SPLIT     a push kernel, then a separate merge kernel after a cross-GPU wait.
 * Results are bit-identical under every schedule.  Errors: CS_ENOTINIT, CS_EINVAL. */
#define CS_SCHED_INSTEP   0
#define CS_SCHED_DEFERRED 1
#define CS_SCHED_SPLIT    2
int cs_set_schedule(int schedule);

/* Test hook: from the next cs_bind (nprocs == 1), run the multi-GPU protocol for
 * `vranks` ranks on this one GPU: rank v owns rows [v*world/vranks, (v+1)*world/vranks)
 * of the bound buffers (which hold all `world` rows), has its own exchange region, and
 * every kernel is one cooperative launch whose CTAs are split among the ranks, so ranks
 * that wait on one another are co-resident.  Same kernels, flags and peer addressing as
 * across GPUs.  vranks = 1 restores the normal binding.  Errors: CS_ENOTINIT, CS_EINVAL. */
int cs_test_emulate_ranks(int vranks);

/* Multi-GPU (nprocs > 1): export this process's peer-visible exchange region
 * (allocated by cs_bind) as a CUDA IPC handle (CS_IPC_HANDLE_BYTES bytes into
 * handle_out).  The caller all-gathers the handles (e.g. over torch.distributed)
 * and passes all nprocs of them, in rank order, to cs_ipc_import, which maps the
 * peers' regions (NVLink peer memory).  Collective in the sense that every
 * process must import before any process steps.
 * Errors: CS_ENOTBOUND, CS_EINVAL, CS_ECUDA. */
int cs_ipc_export(char* handle_out);
int cs_ipc_import(const char* all_handles /* nprocs * CS_IPC_HANDLE_BYTES */);

/* Multi-GPU hierarchical step through the NVSwitch (NVLS): the intra-group gradient average
 * h1 of cs_hier_step (section 3.3 "reduce the gradients in each group";
 * reading C-12) as an in-switch reduction (multimem.ld_reduce) with a multicast store of
 * the group mean (multimem.st), one kernel (k_hier_nvls) instead of the point-to-point
 * reduce-scatter + all-gather.
 *   cs_multicast_bytes  the workspace size this binding needs (after cs_bind).
 *   cs_set_multicast    registers the caller's workspace: uc_base = this GPU's mapping of a
 *                       buffer bound to a multicast object spanning exactly this process's
 *                       hierarchical group (e.g. torch symmetric memory rendezvoused over
 *                       the group), mc_base = the multicast mapping of the same buffer.
 *                       Caller-owned; must stay mapped until cs_set_multicast(NULL, ...) or
 *                       cs_finalize / cs_bind (which forget it).  Every member must register
 *                       before any member steps (the words at the workspace start are
 *                       zeroed here).  NULL uc_base returns to the point-to-point h1.
 *   cs_add_multicast_grads  registers a caller buffer holding gradients that is bound to the
 *                       same group's multicast object: a `grads` row inside it is reduced in
 *                       place, which requires every member to pass `grads` at the same offset
 *                       of its buffer (a training loop's flat gradient buffer); any other
 *                       `grads` is first copied into the workspace.
 * Numerics: the switch sums the members' fp32 values in its own order, so for groups of
 * >= 3 GPUs params match the oracle within the hierarchical tolerance (SURVEY 8(c):
 * norm-wise <= 1e-6) rather than bitwise; groups of 2 stay bitwise.  Members still hold
 * bit-identical replicas.  LARS keeps the point-to-point h1.  k_hier_nvls keeps all its CTAs
 * co-resident (two per SM) for its two group barriers: other work running on the GPU at the
 * same time delays it, bounded by the 20 s wait limit (CS_ETIMEOUT).  Measured slower than the
 * point-to-point h1 for fp32 on this pool: an opt-in.
 * Errors: CS_ENOTBOUND, CS_EINVAL, CS_ELAYOUT (not 256-B / 16-B aligned), CS_EUNSUPPORTED
 * (one process, emulated ranks, groups of one GPU), CS_ECUDA. */
int cs_multicast_bytes(int64_t* bytes_out);
/* Multi-GPU hierarchical step with the intra-group gradient sum done by NCCL (ncclAllReduce
 * over a communicator of the group's GPUs; north_star: "NCCL over NVLink is used only for
 * the intra-group average of hierarchical mode"); the update kernels multiply the sum by
 * fp32(1/|G|) as they load it.  NCCL is loaded at run time (libnccl.so.2).
 *   cs_nccl_unique_id  fills id_out[CS_NCCL_ID_BYTES] (call on the group's first member).
 *   cs_set_hier_nccl   every member of a group passes the same id (collective over the
 *                      group: blocks until all members joined); NULL returns to the
 *                      point-to-point h1.  Replaces a registered multicast workspace.
 * Numerics: NCCL's summation order, so groups of >= 3 GPUs match the oracle within the
 * hierarchical tolerance; groups of 2 bitwise.  LARS keeps the point-to-point h1.
 * Errors: CS_ENOTBOUND, CS_EINVAL, CS_EUNSUPPORTED (no libnccl, one process, emulated ranks,
 * groups of one GPU), CS_ECUDA (NCCL error). */
#define CS_NCCL_ID_BYTES 128
int cs_nccl_unique_id(char* id_out);
int cs_set_hier_nccl(const char* group_id);
int cs_set_multicast(void* uc_base, void* mc_base, int64_t bytes);
int cs_add_multicast_grads(void* uc_base, void* mc_base, int64_t bytes);

/* ---- the hot path --------------------------------------------------------- */

/* One flat Crossover-SGD step at the internal step counter t, then t += 1.
 * Enqueued on the bound stream:
 *   a2  k topologies src_s = Alg.2(seed, t, s) (device-side, no communication)
 *   a3  m_i <- fl(fl(momentum*m_i) + g_i);  y_i <- fl(x_i - fl(lr*m_i))
 *       ("parameter averaging is processed after the gradient is applied",
 *        PAPER.md:122; readings C-8, C-9)
 *   a4  worker i obtains y_{src_s(i)} on segment s (Alg.1 l.4-8):
 *       an HBM read when co-resident, an NVLink peer store when not
 *   a5  x_i[R_s] <- fl(fl(y_i + y_{src_s(i)}) * 0.5)   (Alg.1 l.17)
 *       psw_{i,s} <- fl(fl(psw_{i,s} + psw_{src_s(i),s}) * 0.5)  (C-11)
 *   a6  (if cs_set_diag(1)) consensus distance and mean checksum, fp64.
 *   params  fp32 device [n_loc][ld], updated in place (push-sum numerator x).
 *   grads   fp32 device [n_loc][ld], read only.
 *   psw     fp32 device [n_loc][k] push-sum weights, updated in place (start at 1).
 *   lr, momentum  fp32 scalars.
 * Every output reads only the pre-step snapshot.  Multi-GPU: every
 * process must call with the same t.  On the default schedule (CS_SCHED_INSTEP) params
 * and psw hold the merged x', w' once the step's enqueued work completes; only the opt-in
 * CS_SCHED_DEFERRED leaves a5 to the next step's kernel (then cs_flush or cs_sync before
 * reading params / psw; see cs_set_schedule, cs_flush).  Also: cs_set_topology_kind (SGP graph), cs_set_wire (bf16 wire),
 * cs_set_lars + cs_set_layers (LARS).  Errors: CS_ENOTBOUND, CS_ELAYOUT, CS_EINVAL,
 * CS_ECUDA, CS_ETOPOLOGY, CS_EDIVERGED (from an earlier step), CS_ETIMEOUT,
 * CS_EUNSUPPORTED (a combination listed as such at the setters). */
int cs_gossip_step(float* params, const float* grads, float* psw, float lr, float momentum);

/* End-to-end variant of cs_gossip_step for host-resident gradients: copies
 * grads_host (n_loc x ld fp32, pinned for full speed) into a library-owned
 * device staging buffer, runs one step with diagnostics, copies the two fp64
 * diagnostics into diag_out[2] = {consensus distance, mean checksum} and
 * synchronises the stream.  params / psw stay device-resident. */
int cs_gossip_step_host(float* params, const float* grads_host, float* psw, float lr,
                        float momentum, double* diag_out);

/* End-to-end variant with the step's input and result in HOST memory: the gradients come
 * from grads_host ([n_loc][ld] fp32, pinned for full speed) and the merged params / psw are
 * copied back to params_host_out ([n_loc][ld]) / psw_host_out ([n_loc][k]) before it
 * returns (synchronous).  params / psw / momentum stay the device state of the job.  The
 * vector is cut into 8 column pieces: the host->device copy of piece q+1 and the
 * device->host copy of piece q-1 overlap the step kernel on piece q (copy engines in both
 * directions, k_gossip_tma on a tile range; the last piece mixes the push-sum weights).
 * Single-GPU bulk-TMA path without LARS or diagnostics (CS_EUNSUPPORTED otherwise).
 * Errors as cs_gossip_step, CS_EINVAL (NULL host buffer). */
int cs_gossip_step_io(float* params, const float* grads_host, float* psw, float lr, float momentum,
                      float* params_host_out, float* psw_host_out);

/* One hierarchical step (§3.3) at step t, then t += 1:
 *   h1  per group, gbar = fl(sum_{i in G, ascending} g_i) * fp32(1/|G|)
 *   h2  leaders apply a3 with gbar, then a4/a5 among the G leaders with the
 *       leader topology (tag HIER); G == 1 skips the exchange (x = y)
 *   h3  every member's params and psw become its leader's (bitwise)
 * `grads` is read only.  Momentum is defined at leaders only.
 * One GPU: members' momentum rows are left untouched.
 * Several GPUs (one worker per GPU, world == nprocs): the group's gradient is
 * reduce-scattered over NVLink and summed in ascending member order (so the result
 * is the same bits as on one GPU), every member holds an exact replica of its
 * leader's params, momentum and psw and exchanges with the member of the same index
 * in the source group.  The first hierarchical step after cs_bind / cs_set_step
 * copies each leader's state to its members; callers must not modify a member's
 * state between hierarchical steps.  Other layouts: CS_EUNSUPPORTED.
 * With LARS (cs_set_lars) the leader's rates come from its x and the group-reduced
 * gradient gbar, so the gradient norm is the synchronised one; on
 * several GPUs every member computes the same rates from its replica.  On one GPU
 * cs_get_lars_rates' first `groups` rows are the groups' rates.
 * Errors as cs_gossip_step. */
int cs_hier_step(float* params, float* grads, float* psw, float lr, float momentum);

/* ---- state, diagnostics, test hooks ------------------------------------------ */

/* Communication-interval mode (section 4: "increase the communication
 * interval and accumulate the loss during this interval"; Table 1 "Communication
 * Interval 42"; SPEC accumulate_and_flush).  Micro-step `count`
 * (0 <= count < interval) of an interval of `interval` micro-steps, over the
 * bound [n_loc, ld] rows (columns [0, d); padding columns are never written):
 *   count == 0             acc = 0 + grads            (acc is not read)
 *   0 < count              acc = fl(acc + grads)
 *   count == interval - 1  then acc = fl(acc / interval)   (IEEE division)
 * After the last micro-step acc holds the interval's mean gradient and is passed
 * to cs_gossip_step / cs_hier_step as `grads`: one gossip round per interval.
 * The caller owns both buffers (device, 16-byte aligned, row stride ld) and the
 * count.  Local to each process: no exchange.  Enqueued on the bound stream.
 * Errors: CS_ENOTBOUND, CS_EINVAL (NULL, count outside [0, interval), interval
 * outside [1, 2^24)), CS_ELAYOUT (alignment), CS_ECUDA. */
int cs_accumulate(float* acc, const float* grads, int count, int interval);

/* Layer-aligned segment plan helper (host only; SPEC.md:40-47 build_segment_plan,
 * Table 1 "Segmenting blocks and FC layer").  Partitions n_layers
 * consecutive layers of element counts layer_sizes[] into k contiguous non-empty
 * segments minimising the largest segment; among those, each segment left to right
 * takes as many layers as possible (reading C-19).  Writes seg_of_layer_out[n_layers].
 * Errors: CS_EINVAL (NULL, n_layers outside [1, CS_MAX_LAYERS], a size < 1),
 * CS_EINVAL_SEGMENTS (k outside [1, n_layers]). */
int cs_segment_plan(const int64_t* layer_sizes, int n_layers, int k, int32_t* seg_of_layer_out);

/* Layer table of the bound vector (host arrays, copied): layer l is columns
 * [layer_bounds[l], layer_bounds[l+1]), layer_bounds[0] = 0, layer_bounds[n_layers] = d,
 * strictly increasing, every interior bound a multiple of 4 elements (16-byte rows for
 * bulk copies).  seg_of_layer (may be NULL) assigns the layers to the k segments of
 * cs_init: non-decreasing from 0 to k-1 in steps of 0 or 1; the segment bounds become
 * the layer bounds where it steps (the paper's "blocks and FC layer" plan).  NULL keeps
 * the equal split of reading C-2; the layers then only serve LARS.  layer_bounds NULL
 * or n_layers 0 clears the table.  Lives until the next cs_bind.
 * Runs on the single-GPU bulk-TMA path (world <= 64, k*world <= 2048) and on the
 * multi-GPU paths, push/mix and hybrid walk (every process must pass the same table;
 * synchronises the bound stream), for the flat and the hierarchical step.  The
 * multi-GPU paths refuse it together with the bf16 wire.
 * Errors: CS_ENOTBOUND, CS_EINVAL, CS_ELAYOUT (bounds), CS_EINVAL_SEGMENTS,
 * CS_EUNSUPPORTED (the register path), CS_ECUDA. */
int cs_set_layers(const int64_t* layer_bounds, int n_layers, const int32_t* seg_of_layer);

/* LARS in the flat step ("adapts the learning rate of each layer by the
 * ratio of the weight norm to the gradient norm"; Table 1: eta 0.0025, weight decay
 * 5e-5).  eta > 0 enables, eta == 0 disables.  With it enabled,
 * every flat step computes, for each worker i and layer l, from this step's x and g:
 *   scale = eta*|x_il| / ((|g_il| + wd*|x_il|) + eps)   (fp64; 1 if a norm is 0)
 * (|x_il| of this step's x: recomputed every step unless cs_set_lars_carry(1) is on)
 *   lrs   = fp32(lr * scale)
 * and applies  m = mu*m + (g + wd*x),  y = x - lrs*m  before the exchange (C-18).
 * Needs a layer table at step time (CS_EINVAL otherwise).  Two extra launches per
 * step before the update: k_lars_norms, k_lars_scale (then k_gossip_tma on one GPU,
 * k_peer_push + k_peer_mix or k_hyb_walk + k_hyb_tail across GPUs; the deferred merge is
 * off with LARS because the norms need the merged parameters).
 * Errors: CS_ENOTINIT, CS_EINVAL. */
int cs_set_lars(float eta, float weight_decay, float eps);

/* LARS x-norm carry (opt-in, default off; single-GPU bulk-TMA path).  With it enabled the
 * step kernel also emits each worker's per-tile sums of x'^2, and the next LARS step on the
 * same params buffer takes its ||x|| from them instead of reading x again (24 instead of 28
 * B/param).  The caller then promises that nothing but the library writes params between
 * LARS steps -- or calls cs_params_modified() after it did (a checkpoint load, a manual
 * decay, any in-place op), which makes the next step read x again.  cs_set_step, cs_bind
 * and cs_set_layers also drop the carry.  Errors: CS_ENOTINIT. */
int cs_set_lars_carry(int enable);
int cs_params_modified(void);

/* Rates lrs [n_loc][n_layers] (host, row-major) of the most recent LARS step.
 * Synchronises the stream.  Errors: CS_EINVAL (no LARS step since cs_set_layers). */
int cs_get_lars_rates(float* rates_out);

/* Topology of the flat step (the SGP baseline on the same machinery).
 * CS_TOPO_CROSSOVER: Alg. 2, a fresh load-balanced random derangement per segment
 * (PAPER.md:165-191).  CS_TOPO_EXPONENTIAL: SGP's directed exponential graph
 * ("model-wise communication and directed exponential network topology";
 * SPEC.md:136-144): at step t worker i receives from (i - 2^(t mod log2 world)) mod world,
 * the same peer for every segment (use k = 1 for SGP's model-wise exchange).  The
 * update, merge and push-sum weights are unchanged: halving and pushing to one peer is
 * the merge of Alg. 1 l.17.  Applies to cs_gossip_step, cs_gossip_step_host and
 * cs_topology on every path; the hierarchical step keeps Alg. 2 for its leaders.
 * AllReduce-SGD, the other baseline, is cs_hier_step with groups = 1.
 * Errors: CS_ENOTINIT, CS_EINVAL (unknown kind), CS_EUNSUPPORTED (exponential with a
 * world that is not a power of two), CS_ECUDA. */
int cs_set_topology_kind(int kind);

/* Wire format of the exchanged segments (mixed
 * precision).  CS_WIRE_BF16: every segment a worker receives is the sender's y rounded
 * to the nearest bf16 (ties to even) and widened back exactly; the worker's own y, the
 * momentum, params and push-sum weights stay fp32 (reading C-20):
 *   x'_i = fl(fl(y_i + bf16(y_src(i))) * 0.5)
 * It applies to every received segment, on the same GPU or not, so results do not
 * depend on the placement of workers; across GPUs the inbox holds bf16, halving the
 * NVLink bytes (cs_step_bytes counts 2 B per remote element).  Flat step only (the
 * hierarchical step refuses it).  Takes effect at the next step.
 * Errors: CS_ENOTINIT, CS_EINVAL (unknown format). */
int cs_set_wire(int format);

/* Completes deferred work of earlier steps, enqueued on the bound stream (no host sync).
 * On the multi-GPU push/mix schedule (one worker per GPU) the merge a5 of step t runs
 * inside step t+1's push kernel, tile by tile, before that step's update; this removes
 * a full pass and a cross-GPU wait per step.  Between the two, params hold step t's y
 * and psw its pre-merge weights.  cs_flush, cs_sync, diagnostics, cs_set_step, cs_bind,
 * cs_finalize, LARS and the hierarchical step complete a pending merge first.  Pass the
 * same params/psw buffers to consecutive steps (other buffers flush first).
 * CS_PEER_FUSE=0 in the environment disables the deferral.  Errors: CS_ENOTBOUND, CS_ECUDA. */
int cs_flush(void);

/* Set / read the step counter t (resume = restore buffers + cs_set_step). */
int cs_set_step(int64_t step);
int cs_get_step(int64_t* step_out);

/* Enable (1) / disable (0) the fused diagnostics of later steps (default 0). */
int cs_set_diag(int enable);

/* Diagnostics of the most recent step that had them enabled:
 *   cd_out    = sqrt((1/n) sum_i sum_j (z_ij - zbar_j)^2),  z = x / psw
 *   mean_out  = sum_j zbar_j,   zbar_j = sum_i x_ij / sum_i psw_{i,s(j)}
 * over ALL world workers.  One GPU: fused into the step kernel.  Several GPUs: a
 * pass after the step sends every worker's x' of a column chunk to the chunk's
 * owner GPU and combines the per-GPU partials in rank order (every process gets
 * the same value).  fp64, deterministic.  Synchronises the stream.
 * Errors: CS_EINVAL if no diagnosed step yet, CS_EDIVERGED, CS_ETIMEOUT. */
int cs_get_diag(double* cd_out, double* mean_out);

/* Wait for all enqueued work; reports deferred device errors. */
int cs_sync(void);

/* Test hook: replace the generated topology of the following steps with
 * src [k][world] (receiver -> sender, every row a derangement) until called
 * again with NULL.  Errors: CS_EINVAL_TOPOLOGY. */
int cs_test_set_topology(const int32_t* src);

/* Test hook: run the device topology generator for `step` and copy its
 * [k][world] output to src_out (host).  Synchronises. */
int cs_test_device_topology(int64_t step, int tag, int32_t* src_out);

/* Input generator for tests and the benchmark (NOT part of the method): fills
 * rows [row0, row0+rows) x [0, d) of a device fp32 matrix with row stride ld with
 * scale * H(seed, tag, row, j), the SplitMix64 counter hash of synth/__init__.py.
 * Enqueued on the bound stream (or the legacy stream before cs_bind). */
int cs_synth_fill(float* out, int64_t rows, int64_t d, int64_t ld, uint64_t seed,
                  int tag, int64_t row0, float scale);

/* Bytes per step the hot kernel moves, for roofline accounting:
 * out[0] = algorithmic HBM bytes, out[1] = NVLink bytes into this GPU at step t
 * (exact, from the topology), for flat (hier = 0) or hierarchical (hier = 1).
 * Flat: 20 B per parameter per local worker; with LARS 28 B (the norm pass reads x and
 * g), or 24 B on one GPU once the previous LARS step carried the x norms. */
int cs_step_bytes(int64_t step, int hier, double* out);

/* Kernel timing for roofline accounting: with cs_set_timing(1) every later step
 * records a CUDA event pair on the bound stream around its hot kernel(s)
 * (the names cs_kernel_info returns; with LARS the pair brackets all three launches).  cs_set_timing(1) also
 * clears earlier records.  cs_get_timing synchronises and returns the summed
 * event-measured duration (ms) and the number of timed launches. */
int cs_set_timing(int enable);
int cs_get_timing(double* total_ms_out, int64_t* launches_out);

/* Name of the hot kernel the most recent step launched (static string, "" before
 * the first step) and the number of library kernel launches that step issued. */
const char* cs_kernel_info(int* launches_per_step_out);

#ifdef __cplusplus
}
#endif
#endif /* CROSSOVER_SGD_H */
