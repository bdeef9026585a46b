// Native step loop: Simulation.run / SignalEngine.run_steps (reference
// core.py:262-279) with the rebuild policy of Simulation._compute_forces and
// _rebuild (sim.py:114-149), driven from C++.
//
// Ungraphed step (first / last step of a call, and every step when use_graph = 0):
//     k_integrate      finalize(s-1) + integrate(s) + displacement check
//     64-byte D2H      status block -> pinned host copy, then an event
//     k_force_lj       launched speculatively with the current list
// The host inspects the rebuild flag while the force kernel is running.  In the
// common case (flag clear) nothing else happens and the GPU never idles.  If the
// flag is set, the speculative forces are discarded: (reorder) -> bin -> list
// build -> snapshot, the overflow word is read (one sync per rebuild), and the
// force kernel is launched again on the fresh list.
//
// Graphed step (use_graph = 1, middle steps of a call): one cudaGraphLaunch per MD
// step and no host round trip at all --
//     k_integrate<2, gated> -> k_graph_gate (cudaGraphSetConditional(flag))
//       -> IF node { whole rebuild sequence, k_graph_after_build }
//       -> k_force_lj (gated) -> k_graph_step_done
// Pointers are baked into the graph, so a reorder inside the graph gathers into the
// spare buffers and copies back.  A list build that overflows inside the graph sets
// status->frozen: the remaining launches of the batch return immediately, the host
// reads how many steps really completed and continues exactly like the ungraphed
// overflow case (grow the stride, rebuild, resume the interrupted step).
#include <algorithm>
#include <new>
#include <vector>

#include "common.cuh"

using namespace b2md;

struct b2md_runner {
    b2md_runner_config cfg;
    std::vector<double> table;
    b2md_grid grid;
    double r_list;
    double half_skin2;
    int current;
    bool pending_kick;        // finalize of the previous step not applied yet
    bool list_valid;
    bool mid_step;            // stopped after integrate, before a successful rebuild
    int rebuilds_total;
    b2md_status *h_status;    // pinned
    cudaEvent_t ev;           // flag read-back
    cudaEvent_t ev_in;        // ordering against the caller's stream
    cudaStream_t stream;      // the runner's own (capturable) stream
    cudaStream_t copy_stream; // flag read-backs, off the kernels' critical path
    bool own_h_status, own_stream, own_copy_stream;   // false: lent by the caller (cfg)
    cudaEvent_t ev_mark;      // "everything enqueued so far" for the copy stream
    int64_t launches;
    double last_disp2;        // max squared displacement seen one step ago (fp32 check)
    // step graphs: [0] = one MD step, [1] = steps_per_graph MD steps
    cudaGraph_t graph[2];
    cudaGraphExec_t graph_exec[2];
    int steps_per_graph;
    int64_t graph_launch_kernels;   // kernels per step in the always-executed part
    int64_t graph_rebuild_kernels;  // kernels inside one conditional body
    // The host-launched rebuild sequence (~25 small kernels) as one graph launch per live-set
    // parity: at N <= 10^5 the sequence is launch-bound (250 us of launches for 60 us of work)
    cudaGraphExec_t rebuild_exec[2];
    int64_t rebuild_exec_kernels[2];
    int rebuild_seen[2];            // host-launched rebuilds per parity (a graph pays from the 2nd on)
    // one-launch steps (b2md_force_lj_pairs_advance)
    void *pos_cur;            // where the live position high words are (canonical or alt)
    bool ahead;               // positions already advanced to the step about to be processed
    int gate_in;              // status word holding the rebuild flag of those positions
    int count_seen;           // advance launches counted by the device so far (word 13)
    // velocities uploaded on a side stream (cfg.vel_ready_event): the first build gathers
    // them last, behind the list build, so that the upload overlaps it
    bool defer_vel, vel_waited;
    // pruned pair rows (cfg.prune_delta > 0): what the next one-launch step may walk
    bool prune_on;
    int inner_state;          // kInnerNeedPrune / kInnerValid / kInnerOuterOnly
    bool after_integrate;     // positions came from k_integrate: inner flags unknown for them
    int steps_since_prune;
    bool refreshed;           // the late refresh of this list's inner rows has been tried
    int64_t prunes_total, outer_steps_total;
    // Andersen thermostat (second finalize slot of the reference, sim.py:86-87)
    double thermo_p, thermo_t;
    uint64_t thermo_seed;
    int64_t first_step;       // SignalEngine.step_count of the first step of the next run
    // phase timers: GPU time of a call and of its rebuild sequences (CUDA events)
    cudaEvent_t ev_run[2];
    std::vector<cudaEvent_t> ev_rebuild;   // pairs, grown on demand, resolved at the end of a call
    int rebuild_events_used;
};

namespace {

struct Set {
    void *pos_hi, *pos_lo, *vel, *force, *image;
    float *virial;
};

Set buffer_set(const b2md_runner *r, int k) {
    const b2md_runner_config &c = r->cfg;
    return Set{c.pos_hi[k], c.pos_lo[k], c.vel[k], c.force[k], c.image[k], c.virial[k]};
}
Set live(const b2md_runner *r) { return buffer_set(r, r->current); }
Set spare(const b2md_runner *r) { return buffer_set(r, 1 - r->current); }

int stride_rows(const b2md_runner *r) {
    const int m = r->cfg.list_row_multiple > 0 ? r->cfg.list_row_multiple : 16;
    return (r->cfg.stride + m - 1) / m * m;
}

__global__ void k_graph_gate(cudaGraphConditionalHandle handle, const b2md_status *status) {
    const bool go = !status->frozen && status->rebuild_flag != 0;
    cudaGraphSetConditional(handle, go ? 1u : 0u);
}

__global__ void k_graph_after_build(b2md_status *status) {
    status->graph_rebuilds += 1;
    if (status->overflow) status->frozen = 1;
}

__global__ void k_graph_step_done(b2md_status *status) {
    if (!status->frozen) status->graph_steps += 1;
}

__global__ void k_graph_batch_reset(b2md_status *status) {
    status->graph_steps = 0;
    status->graph_rebuilds = 0;
    status->frozen = 0;
}

int read_status(b2md_runner *r) {
    int rc = check_cuda(cudaMemcpyAsync(r->h_status, r->cfg.status, sizeof(b2md_status),
                                        cudaMemcpyDeviceToHost, r->stream), "status read-back");
    if (rc) return rc;
    return check_cuda(cudaStreamSynchronize(r->stream), "status sync");
}

// b2md_runner_config::pair_schedule: bit 0 block schedule, bit 1 lane order
int pair_flags(const b2md_runner_config &c) {
    if (c.pair_rows <= 0) return 0;
    return ((c.pair_schedule & 1) ? B2MD_FORCE_SCHEDULED : 0) |
           ((c.pair_schedule & 2) ? B2MD_FORCE_ORDERED : 0);
}

// thermo = false on steps whose per-particle energies cannot be observed
int launch_force(b2md_runner *r, bool thermo, bool gated = false) {
    const b2md_runner_config &c = r->cfg;
    Set a = live(r);
    r->launches += 1;
    const int flags = (thermo ? 0 : B2MD_FORCE_SKIP_THERMO) | (gated ? B2MD_FORCE_GATED : 0) |
                      pair_flags(c);
    if (c.pair_rows > 0)
        return b2md_force_lj_pairs(a.pos_hi, c.n, &c.box, c.pair_nbr, c.pair_counts,
                                   c.pair_pitch, c.nbr, c.counts, c.pitch, c.boundary,
                                   r->table.data(), c.ntypes, flags, a.force, a.virial, c.status,
                                   r->stream);
    return b2md_force_lj(a.pos_hi, c.n, &c.box, c.nbr, c.counts, c.pitch, stride_rows(r),
                         c.boundary, r->table.data(), c.ntypes, flags, a.force, a.virial,
                         c.status, r->stream);
}

constexpr int kWordRebuildFlag = 5;   // b2md_status::rebuild_flag
constexpr int kWordAltFlag = 12;      // b2md_status::reserved[0]
constexpr int kWordAdvanceCount = 13; // b2md_status::reserved[1]
constexpr int kWordThirdFlag = 14;    // b2md_status::reserved[2]: pruned loops rotate three words
constexpr int kInnerNeedPrune = 0, kInnerValid = 1, kInnerOuterOnly = 2;

// Gate word after `w`: two words alternate in the plain loop; with pruned pair rows the flag
// bits do not clear themselves, so three words rotate (b2md_force_lj_pairs_advance_pruned).
int next_gate(const b2md_runner *r, int w) {
    if (!r->prune_on) return w == kWordRebuildFlag ? kWordAltFlag : kWordRebuildFlag;
    return w == kWordRebuildFlag ? kWordAltFlag : (w == kWordAltFlag ? kWordThirdFlag : kWordRebuildFlag);
}

bool thermostatted(const b2md_runner *r) { return r->thermo_p > 0.0; }

bool can_advance(const b2md_runner *r) {
    const b2md_runner_config &c = r->cfg;
    return c.pos_hi_alt != nullptr && c.use_graph == 0 && !thermostatted(r);
}

// The canonical buffer of the live set holds the position high words again.
int canonicalize(b2md_runner *r) {
    Set a = live(r);
    if (r->pos_cur == nullptr || r->pos_cur == a.pos_hi) { r->pos_cur = a.pos_hi; return 0; }
    int rc = check_cuda(cudaMemcpyAsync(a.pos_hi, r->pos_cur, 16 * (size_t)r->cfg.n,
                                        cudaMemcpyDeviceToDevice, r->stream), "position copy");
    r->pos_cur = a.pos_hi;
    return rc;
}

// force(s) + finalize(s) + integrate(s+1) in one launch, gated on the rebuild flag of
// the positions it reads; the advanced high words go to the other buffer.
int launch_advance(b2md_runner *r, int prune_mode = 0) {
    const b2md_runner_config &c = r->cfg;
    Set a = live(r);
    void *in = r->pos_cur ? r->pos_cur : a.pos_hi;
    void *out = in == a.pos_hi ? c.pos_hi_alt : a.pos_hi;
    const int gate_out = next_gate(r, r->gate_in);
    r->launches += 1;
    if (prune_mode)
        return b2md_force_lj_pairs_advance_pruned(
            in, out, a.pos_lo, a.vel, a.image, c.n, &c.box, c.dt, c.ref_pos, r->half_skin2,
            c.pair_nbr, c.pair_counts, c.pair_pitch, c.nbr, c.counts, c.pitch, c.boundary,
            r->table.data(), c.ntypes, pair_flags(c), r->gate_in,
            gate_out, next_gate(r, gate_out), prune_mode, c.pair_nbr_inner, c.pair_counts_inner,
            c.pair_rows, c.r_cut, c.skin, c.prune_delta, c.status, r->stream);
    if (c.pair_rows <= 0)
        return b2md_force_lj_advance(in, out, a.pos_lo, a.vel, a.image, c.n, &c.box, c.dt,
                                     c.ref_pos, r->half_skin2, c.nbr, c.counts, c.pitch,
                                     stride_rows(r), c.boundary, r->table.data(), c.ntypes, 0,
                                     r->gate_in, gate_out, c.status, r->stream);
    return b2md_force_lj_pairs_advance(in, out, a.pos_lo, a.vel, a.image, c.n, &c.box, c.dt,
                                       c.ref_pos, r->half_skin2, c.pair_nbr, c.pair_counts,
                                       c.pair_pitch, c.nbr, c.counts, c.pitch, c.boundary,
                                       r->table.data(), c.ntypes,
                                       pair_flags(c), r->gate_in,
                                       gate_out, c.status, r->stream);
}

int reorder_key_bits(const b2md_runner *r) {
    const b2md_runner_config &c = r->cfg;
    if (c.reorder_mode == 1) return b2md_hilbert_key_bits(&r->grid, c.hilbert_bits);
    int key_bits = 1;
    while ((1ll << key_bits) < r->grid.n_cells) ++key_bits;
    return key_bits;
}

// Enqueue key generation, sort and row gathers.  write_back = false: the spare set
// becomes the live one (pointer swap); write_back = true: rows are copied back so
// that the live pointers never change (needed inside a captured graph).
int enqueue_reorder(b2md_runner *r, bool write_back, int64_t *kernels) {
    const b2md_runner_config &c = r->cfg;
    Set a = live(r), b = spare(r);
    cudaStream_t s = r->stream;
    int rc;
    const int key_bits = reorder_key_bits(r);
    if (key_bits < 0) { set_error("reorder: Hilbert key does not fit"); return -5; }
    if (c.reorder_mode == 1) {
        rc = b2md_hilbert_keys(a.pos_hi, a.pos_lo, c.n, &r->grid, c.hilbert_bits, c.keys, s);
    } else {
        // cell order needs the cell of every particle first
        rc = b2md_bin(a.pos_hi, a.pos_lo, c.n, &r->grid, c.cell_of, c.cell_start,
                      c.cell_particles, c.bin_scratch, s);
        *kernels += 3 + scan_launches(r->grid.n_cells);
        if (rc) return rc;
        rc = b2md_cell_keys(c.cell_of, c.n, c.keys, s);
    }
    if (rc) return rc;
    if ((rc = b2md_iota_i32(c.perm, c.n, s))) return rc;
    if ((rc = b2md_sort_pairs_u64(c.keys, c.perm, c.keys_tmp, c.perm_tmp, c.n, key_bits,
                                  c.sort_scratch, s))) return rc;
    *kernels += 2 + ((key_bits + 7) / 8) * (2 + scan_launches(256 * ((c.n + 1023) / 1024)));
    if (r->defer_vel && !write_back) {
        // first build of a runner whose velocities are still arriving over PCIe: only what
        // the list build needs now; enqueue_rebuild gathers the velocities behind it (forces
        // and virial hold nothing yet: b2md_runner_prepare evaluates them on the new rows)
        if ((rc = b2md_gather16(a.pos_hi, b.pos_hi, c.perm, c.n, s))) return rc;
        if ((rc = b2md_gather16(a.pos_lo, b.pos_lo, c.perm, c.n, s))) return rc;
        if ((rc = b2md_gather16(a.image, b.image, c.perm, c.n, s))) return rc;
        *kernels += 3;
    } else {
        const void *src[5] = {a.pos_hi, a.pos_lo, a.vel, a.force, a.image};
        void *dst[5] = {b.pos_hi, b.pos_lo, b.vel, b.force, b.image};
        if ((rc = b2md_gather_rows(src, dst, a.virial, b.virial, c.perm, c.n, s))) return rc;
        *kernels += 1;
    }
    if (write_back) {
        const size_t row = 16 * (size_t)c.n;
        void *dst[5] = {a.pos_hi, a.pos_lo, a.vel, a.force, a.image};
        void *src[5] = {b.pos_hi, b.pos_lo, b.vel, b.force, b.image};
        for (int k = 0; k < 5; ++k)
            if ((rc = check_cuda(cudaMemcpyAsync(dst[k], src[k], row, cudaMemcpyDeviceToDevice, s),
                                 "reorder copy-back"))) return rc;
        if ((rc = check_cuda(cudaMemcpyAsync(a.virial, b.virial, 4 * (size_t)c.n,
                                             cudaMemcpyDeviceToDevice, s), "reorder copy-back")))
            return rc;
    } else {
        r->current = 1 - r->current;
    }
    return 0;
}

// (reorder) -> status reset -> bin -> build -> snapshot, nothing synchronous.
int enqueue_rebuild(b2md_runner *r, bool do_reorder, bool write_back, int64_t *kernels) {
    const b2md_runner_config &c = r->cfg;
    cudaStream_t s = r->stream;
    int rc;
    if (do_reorder && (rc = enqueue_reorder(r, write_back, kernels))) return rc;
    Set a = live(r);
    if ((rc = b2md_status_reset_list(c.status, s))) return rc;
    if ((rc = b2md_bin(a.pos_hi, a.pos_lo, c.n, &r->grid, c.cell_of, c.cell_start,
                       c.cell_particles, c.bin_scratch, s))) return rc;
    // an overflowed list is never used here: the caller grows the stride and rebuilds
    if (c.pair_rows > 0) {
        // list and pair rows in one go (the plain rows are written only where a pair straddles
        // two cells)
        if ((rc = b2md_build_pair_list(a.pos_hi, a.pos_lo, c.n, &c.box, &r->grid, c.cell_of,
                                       c.cell_start, c.cell_particles, r->r_list, c.stride,
                                       c.pitch, c.nbr, c.counts, c.boundary, r->r_list + c.skin,
                                       c.n, B2MD_LIST_ANY_PREFIX, stride_rows(r), c.pair_nbr,
                                       c.pair_counts, c.pair_pitch, c.pair_rows, c.status, s)))
            return rc;
    } else if ((rc = b2md_build_nlist_ex(a.pos_hi, a.pos_lo, c.n, &c.box, &r->grid, c.cell_of,
                                         c.cell_start, c.cell_particles, r->r_list, c.stride,
                                         c.pitch, c.nbr, c.counts, c.boundary, r->r_list + c.skin,
                                         c.n, B2MD_LIST_ANY_PREFIX, c.status, s))) {
        return rc;
    }
    if ((rc = b2md_snapshot(a.pos_hi, a.pos_lo, a.image, c.n, &c.box, c.at_build, c.ref_pos, s)))
        return rc;
    *kernels += 1 + 3 + scan_launches(r->grid.n_cells) + 2 + 1;
    if (c.pair_rows > 0) {
        *kernels += 1;
        if (c.pair_schedule & 1) {
            if ((rc = b2md_pair_schedule(c.boundary, c.n, c.pair_counts, c.pair_pitch, s)))
                return rc;
            *kernels += 2;
        }
        if (c.pair_schedule & 2) {
            const int unit = (c.pair_schedule >> 8) & 63;
            if ((rc = b2md_pair_order(c.boundary, c.n, c.pair_nbr, c.pair_counts, c.pair_pitch,
                                      c.pair_rows, unit ? unit : 1, (c.pair_schedule >> 2) & 1, s)))
                return rc;
            *kernels += 1;
        }
    }
    if (r->defer_vel && !write_back) {
        // the velocities: wait for their upload, then bring them into the new row order
        if ((rc = check_cuda(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(c.vel_ready_event), 0),
                             "velocity upload wait"))) return rc;
        if (do_reorder) {
            Set now = live(r), old = spare(r);         // (enqueue_reorder swapped the sets)
            if ((rc = b2md_gather16(old.vel, now.vel, c.perm, c.n, s))) return rc;
            *kernels += 1;
        }
        r->defer_vel = false;
        r->vel_waited = true;
    }
    return 0;
}

// Ungraphed rebuild: enqueue, then read overflow / max_count (one sync).
int rebuild(b2md_runner *r, b2md_run_report *rep) {
    const b2md_runner_config &c = r->cfg;
    const bool do_reorder = c.reorder_mode != 0 && (r->rebuilds_total % c.reorder_every) == 0;
    // phase timer: one event pair per rebuild, read when the call ends
    if ((size_t)r->rebuild_events_used + 2 > r->ev_rebuild.size()) {
        for (int k = 0; k < 2; ++k) {
            cudaEvent_t e = nullptr;
            int rc0 = check_cuda(cudaEventCreate(&e), "cudaEventCreate");
            if (rc0) return rc0;
            r->ev_rebuild.push_back(e);
        }
    }
    cudaEvent_t ev0 = r->ev_rebuild[r->rebuild_events_used];
    cudaEvent_t ev1 = r->ev_rebuild[r->rebuild_events_used + 1];
    int rc = check_cuda(cudaEventRecord(ev0, r->stream), "rebuild timer");
    if (rc) return rc;
    // graph mode keeps the live pointers fixed (they are baked into the step graph)
    // (instantiating a graph costs about as much as launching the sequence once: the first
    // rebuild of each parity is launched directly, so that short runs do not pay for it)
    const bool as_graph = c.use_graph == 0 && (c.reorder_mode == 0 || c.reorder_every == 1) &&
                          r->rebuild_seen[r->current]++ > 0 &&
                          env_choice("B2MD_REBUILD_GRAPH", 1) != 0;
    if (as_graph) {
        // one captured sequence per parity of the live set (a reorder flips the sets, so the
        // pointers differ); replayed with a single launch from then on
        const int parity = r->current;
        if (!r->rebuild_exec[parity]) {
            cudaGraph_t graph = nullptr;
            int64_t kernels = 0;
            if ((rc = check_cuda(cudaStreamBeginCapture(r->stream, cudaStreamCaptureModeRelaxed),
                                 "rebuild capture"))) return rc;
            const int rc_enq = enqueue_rebuild(r, do_reorder, false, &kernels);
            const int rc_end = check_cuda(cudaStreamEndCapture(r->stream, &graph), "rebuild capture end");
            r->current = parity;                       // the capture only recorded: undo the flip
            if (rc_enq) { if (graph) cudaGraphDestroy(graph); return rc_enq; }
            if (rc_end) return rc_end;
            rc = check_cuda(cudaGraphInstantiate(&r->rebuild_exec[parity], graph, 0),
                            "rebuild graph instantiate");
            cudaGraphDestroy(graph);
            if (rc) return rc;
            r->rebuild_exec_kernels[parity] = kernels;
        }
        if ((rc = check_cuda(cudaGraphLaunch(r->rebuild_exec[parity], r->stream), "rebuild graph")))
            return rc;
        r->launches += r->rebuild_exec_kernels[parity];
        if (do_reorder) r->current = 1 - r->current;
    } else {
        rc = enqueue_rebuild(r, do_reorder, c.use_graph != 0, &r->launches);
        if (rc) return rc;
    }
    if ((rc = check_cuda(cudaEventRecord(ev1, r->stream), "rebuild timer"))) return rc;
    r->rebuild_events_used += 2;
    if (do_reorder) rep->reorders += 1;
    r->rebuilds_total += 1;
    rep->rebuilds += 1;
    if ((rc = read_status(r))) return rc;
    rep->max_count = r->h_status->max_count;
    rep->n_boundary = r->h_status->n_boundary;
    r->list_valid = r->h_status->overflow == 0;
    r->pos_cur = live(r).pos_hi;      // callers hand over canonical positions; sets may swap
    r->count_seen = 0;                // the status reset of the rebuild cleared the counter
    r->inner_state = kInnerNeedPrune; // new outer rows: the inner ones are void
    r->after_integrate = false;       // (the list snapshot is these positions)
    r->refreshed = false;
    return 0;
}

void destroy_graph(b2md_runner *r) {
    for (int g = 0; g < 2; ++g) {
        if (r->rebuild_exec[g]) cudaGraphExecDestroy(r->rebuild_exec[g]);
        r->rebuild_exec[g] = nullptr;
        r->rebuild_seen[g] = 0;
    }
    for (int g = 0; g < 2; ++g) {
        if (r->graph_exec[g]) cudaGraphExecDestroy(r->graph_exec[g]);
        if (r->graph[g]) cudaGraphDestroy(r->graph[g]);
        r->graph_exec[g] = nullptr;
        r->graph[g] = nullptr;
    }
}

// Capture `n_steps` MD steps (fused integrate, conditional rebuild, no-thermo
// force) into graph slot `slot`.  Every step gets its own conditional handle and
// its own copy of the rebuild body.
int build_graph(b2md_runner *r, int slot, int n_steps) {
    const b2md_runner_config &c = r->cfg;
    cudaStream_t s = r->stream;
    int rc;
    if ((rc = check_cuda(cudaGraphCreate(&r->graph[slot], 0), "cudaGraphCreate"))) return rc;
    cudaGraph_t graph = r->graph[slot];
    std::vector<cudaGraph_t> bodies(n_steps, nullptr);
    int64_t main_kernels = 0, body_kernels = 0;
    if ((rc = check_cuda(cudaStreamBeginCaptureToGraph(s, graph, nullptr, nullptr, 0,
                                                       cudaStreamCaptureModeRelaxed),
                         "begin capture"))) return rc;
    Set a = live(r);
    for (int k = 0; k < n_steps && !rc; ++k) {
        cudaGraphConditionalHandle handle;
        rc = check_cuda(cudaGraphConditionalHandleCreate(&handle, graph, 0,
                                                         cudaGraphCondAssignDefault),
                        "cudaGraphConditionalHandleCreate");
        if (rc) break;
        rc = b2md_vv_integrate_gated(a.pos_hi, a.pos_lo, a.vel, a.force, a.image, c.n, &c.box,
                                     c.dt, c.ref_pos, r->half_skin2, c.status, 2, s);
        if (rc) break;
        k_graph_gate<<<1, 1, 0, s>>>(handle, c.status);
        // splice the conditional node in after what has been captured so far
        cudaStreamCaptureStatus cap_status;
        cudaGraph_t cap_graph = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t n_deps = 0;
        cudaGraphNode_t cond_node = nullptr;
        rc = check_cuda(cudaStreamGetCaptureInfo(s, &cap_status, nullptr, &cap_graph, &deps,
                                                 &n_deps), "capture info");
        if (rc) break;
        cudaGraphNodeParams params = {};
        params.type = cudaGraphNodeTypeConditional;
        params.conditional.handle = handle;
        params.conditional.type = cudaGraphCondTypeIf;
        params.conditional.size = 1;
        rc = check_cuda(cudaGraphAddNode(&cond_node, graph, deps, n_deps, &params),
                        "add conditional node");
        if (rc) break;
        bodies[k] = params.conditional.phGraph_out[0];
        rc = check_cuda(cudaStreamUpdateCaptureDependencies(s, &cond_node, 1,
                                                            cudaStreamSetCaptureDependencies),
                        "update capture dependencies");
        if (rc) break;
        rc = launch_force(r, false, true);
        r->launches -= 1;    // only captured, not launched
        if (rc) break;
        k_graph_step_done<<<1, 1, 0, s>>>(c.status);
    }
    main_kernels = 4;
    cudaGraph_t ended = nullptr;
    int rc_end = check_cuda(cudaStreamEndCapture(s, &ended), "end capture");
    if (rc) return rc;
    if (rc_end) return rc_end;

    // bodies of the IF nodes: the whole rebuild, captured on the same stream
    for (int k = 0; k < n_steps; ++k) {
        cudaGraph_t body = bodies[k];
        body_kernels = 0;
        if ((rc = check_cuda(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                                           cudaStreamCaptureModeRelaxed),
                             "begin body capture"))) return rc;
        rc = enqueue_rebuild(r, c.reorder_mode != 0, true, &body_kernels);
        if (!rc) { k_graph_after_build<<<1, 1, 0, s>>>(c.status); body_kernels += 1; }
        rc_end = check_cuda(cudaStreamEndCapture(s, &ended), "end body capture");
        if (rc) return rc;
        if (rc_end) return rc_end;
    }
    if ((rc = check_cuda(cudaGraphInstantiate(&r->graph_exec[slot], graph, 0),
                         "graph instantiate"))) return rc;
    r->graph_launch_kernels = main_kernels;
    r->graph_rebuild_kernels = body_kernels;
    return 0;
}

// Every path that ends a call has drained the stream (read_status) before it gets here.
void finish_report(b2md_runner *r, b2md_run_report *rep, int64_t launches_before) {
    rep->current = r->current;
    rep->kernel_launches = r->launches - launches_before;
    rep->list_valid = r->list_valid ? 1 : 0;
    if (cudaEventRecord(r->ev_run[1], r->stream) == cudaSuccess &&
        cudaEventSynchronize(r->ev_run[1]) == cudaSuccess) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r->ev_run[0], r->ev_run[1]) == cudaSuccess)
            rep->gpu_ms = ms;
        for (int k = 0; k + 1 < r->rebuild_events_used; k += 2)
            if (cudaEventElapsedTime(&ms, r->ev_rebuild[k], r->ev_rebuild[k + 1]) == cudaSuccess)
                rep->rebuild_gpu_ms += ms;
    }
    (void)cudaGetLastError();      // a timer that could not be read is not an error of the run
    r->rebuild_events_used = 0;
}

// Start of a call: phase timers.
int begin_call(b2md_runner *r) {
    r->rebuild_events_used = 0;
    return check_cuda(cudaEventRecord(r->ev_run[0], r->stream), "run timer");
}

// Second half-kick and the thermostat slot of step number `step` (sim.py:100-102).
// The finalize slots of a thermostatted step (sim.py:86-87: vv_finalize, then the thermostat)
// in one launch; with integrate_next the same pass also integrates the next step (the runner
// is then "ahead", exactly as after b2md_vv_integrate).  Bit-identical to the separate launches.
int finish_thermostat_step(b2md_runner *r, int64_t step, bool integrate_next = false) {
    const b2md_runner_config &c = r->cfg;
    Set a = live(r);
    const int rc = b2md_vv_finalize_andersen(a.pos_hi, a.pos_lo, a.vel, a.force, a.image, c.n,
                                             &c.box, c.dt, r->thermo_seed, (uint64_t)step,
                                             r->thermo_p, r->thermo_t, integrate_next ? 1 : 0,
                                             integrate_next ? c.ref_pos : nullptr, r->half_skin2,
                                             c.status, r->stream);
    r->launches += 1;
    r->pending_kick = false;
    if (integrate_next) {
        r->ahead = true;
        r->gate_in = kWordRebuildFlag;
    }
    return rc;
}

// Make the runner's stream wait for everything the caller enqueued so far.
int order_after_caller(b2md_runner *r) {
    cudaStream_t caller = as_stream(r->cfg.stream);
    int rc = check_cuda(cudaEventRecord(r->ev_in, caller), "order event record");
    if (rc) return rc;
    return check_cuda(cudaStreamWaitEvent(r->stream, r->ev_in, 0), "order stream wait");
}

void toggle_advance_state(b2md_runner *r);

// One ungraphed step.  *stop = 1 when the call must return (overflow / singular).
// With pair rows and a second position buffer the intermediate (unobservable) steps are
// one gated launch each: force(s) + finalize(s) + integrate(s+1) + displacement check.
int plain_step(b2md_runner *r, b2md_run_report *rep, bool thermo, int64_t before, int *stop) {
    const b2md_runner_config &c = r->cfg;
    cudaStream_t s = r->stream;
    Set a = live(r);
    int rc;
    *stop = 0;
    const bool fuse = can_advance(r) && !thermo;
    if (!r->ahead) {
        // positions of this step: integrate in place (canonical buffer)
        if ((rc = canonicalize(r))) return rc;
        if (r->prune_on) {
            // the gate rotation restarts at the rebuild-flag word: all three words clean
            int32_t *w = reinterpret_cast<int32_t *>(c.status);
            const int words[3] = {kWordRebuildFlag, kWordAltFlag, kWordThirdFlag};
            for (int k = 0; k < 3; ++k)
                if ((rc = check_cuda(cudaMemsetAsync(w + words[k], 0, sizeof(int32_t), s),
                                     "gate reset"))) return rc;
            r->after_integrate = true;
        }
        if (r->pending_kick)
            rc = b2md_vv_finalize_integrate(a.pos_hi, a.pos_lo, a.vel, a.force, a.image, c.n,
                                            &c.box, c.dt, c.ref_pos, r->half_skin2, c.status, s);
        else
            rc = b2md_vv_integrate(a.pos_hi, a.pos_lo, a.vel, a.force, a.image, c.n, &c.box, c.dt,
                                   c.ref_pos, r->half_skin2, c.status, s);
        if (rc) return rc;
        r->launches += 1;
        r->gate_in = kWordRebuildFlag;
    }
    r->pending_kick = false;
    // a force evaluation that is observable reads the canonical buffer
    if (!fuse && (rc = canonicalize(r))) return rc;
    // The 64-byte status block travels on a second stream: it waits for what is enqueued
    // so far, but the kernel enqueued next does not wait for the copy.  (That kernel may
    // already update the block while it is being copied: it never touches the flag word
    // read here, and a displacement maximum that is one step ahead only feeds heuristics.)
    if ((rc = check_cuda(cudaEventRecord(r->ev_mark, s), "mark record"))) return rc;
    if ((rc = check_cuda(cudaStreamWaitEvent(r->copy_stream, r->ev_mark, 0), "copy wait"))) return rc;
    if ((rc = check_cuda(cudaMemcpyAsync(r->h_status, c.status, sizeof(b2md_status),
                                         cudaMemcpyDeviceToHost, r->copy_stream),
                         "flag read-back"))) return rc;
    if ((rc = check_cuda(cudaEventRecord(r->ev, r->copy_stream), "event record"))) return rc;
    // Launch the force kernel before the flag is known.  The one-launch step gates
    // itself on the flag; the plain force kernel is skipped when the displacement was
    // already close to the threshold one step ago (a rebuild is likely and waiting a few
    // microseconds beats discarding a force evaluation).
    const bool speculate = fuse || r->last_disp2 < 0.85 * r->half_skin2;
    int mode = 0;
    if (fuse && r->prune_on) {
        const double legal = 0.5 * (c.skin - c.prune_delta);
        if (r->after_integrate || r->inner_state == kInnerOuterOnly) mode = B2MD_PRUNE_OUTER;
        else if (r->inner_state == kInnerNeedPrune) mode = B2MD_PRUNE_NOW;
        // refresh the inner rows while that is still legal: the last prune of a list's life
        // should come as late as the outer rows allow
        else if (!r->refreshed && r->steps_since_prune >= 3 &&
                 r->last_disp2 > 0.78 * legal * legal && r->last_disp2 < 0.98 * legal * legal) {
            mode = B2MD_PRUNE_NOW;
            r->refreshed = true;
        } else mode = B2MD_PRUNE_INNER;
    }
    if (fuse) rc = launch_advance(r, mode);
    else if (speculate) rc = launch_force(r, thermo);
    if (rc) return rc;
    if ((rc = check_cuda(cudaEventSynchronize(r->ev), "event sync"))) return rc;
    rep->max_disp2 = (double)__builtin_bit_cast(float, r->h_status->max_disp2_bits);
    r->last_disp2 = rep->max_disp2;
    if (r->h_status->singular != ~0ull) {
        // a force evaluation of an earlier step met a coincident pair
        // (forces.py:113-116); stop after draining the stream
        if ((rc = read_status(r))) return rc;
        bool stepped = !fuse;
        if (fuse) {
            // the queued launch advanced the particles only if it was not gated out (a
            // rebuild may have been due as well): the device counted it if it ran
            const int ran = reinterpret_cast<const int32_t *>(r->h_status)[kWordAdvanceCount] -
                            r->count_seen;
            if (ran > 0) {
                r->count_seen += ran;
                toggle_advance_state(r);
                r->ahead = true;
                stepped = true;
            }
            // leave the canonical buffer current
            if ((rc = canonicalize(r))) return rc;
            if ((rc = check_cuda(cudaStreamSynchronize(r->stream), "position copy"))) return rc;
        }
        rep->singular = r->h_status->singular;
        rep->reason = B2MD_RUN_SINGULAR;
        r->pending_kick = !fuse;
        if (stepped) rep->steps_done += 1;
        finish_report(r, rep, before);
        *stop = 1;
        return 0;
    }
    const int gate_word = reinterpret_cast<const int32_t *>(r->h_status)[r->gate_in];
    // (pruned loops: bits 2 and 4 of the word are about the inner rows, see launch_advance)
    const bool need_rebuild = r->prune_on ? (gate_word & 1) != 0 : gate_word != 0;
    if (need_rebuild) {
        if (!fuse && speculate) rep->wasted_force_launches += 1;   // (a gated launch did nothing)
        if ((rc = canonicalize(r))) return rc;
        if ((rc = rebuild(r, rep))) return rc;
        r->pos_cur = live(r).pos_hi;          // a reorder may have swapped the sets
        r->gate_in = kWordRebuildFlag;        // both flag words were cleared
        r->last_disp2 = 0.0;
        if (!r->list_valid) {
            r->mid_step = true;
            r->ahead = false;
            rep->reason = B2MD_RUN_OVERFLOW;
            finish_report(r, rep, before);
            *stop = 1;
            return 0;
        }
        if (fuse) {
            mode = r->prune_on ? B2MD_PRUNE_NOW : 0;
            rc = launch_advance(r, mode);
        } else {
            rc = launch_force(r, thermo);
        }
        if (rc) return rc;
    } else if (!speculate) {
        if ((rc = launch_force(r, thermo))) return rc;
    } else if (fuse && mode && ((mode == B2MD_PRUNE_INNER && (gate_word & 2)) ||
                                (mode == B2MD_PRUNE_NOW && (gate_word & 4)))) {
        // the launch found its rows stale (or the prune illegal), returned at once and copied
        // the flags to its output word: clean that word and launch what the flags allow
        if (mode == B2MD_PRUNE_NOW && !(gate_word & 2) && r->inner_state == kInnerValid)
            mode = B2MD_PRUNE_INNER;                        // the refresh came too late: carry on
        else if (!(gate_word & 4)) mode = B2MD_PRUNE_NOW;
        else { mode = B2MD_PRUNE_OUTER; r->inner_state = kInnerOuterOnly; }
        if ((rc = check_cuda(cudaMemsetAsync(reinterpret_cast<int32_t *>(c.status) +
                                                 next_gate(r, r->gate_in), 0, sizeof(int32_t), s),
                             "gate clean"))) return rc;
        r->launches -= 1;                                   // (the gated launch did nothing)
        if ((rc = launch_advance(r, mode))) return rc;
    }
    if (fuse && mode) {
        if (mode == B2MD_PRUNE_NOW) {
            r->inner_state = kInnerValid;
            r->steps_since_prune = 0;
            r->prunes_total += 1;
        } else {
            r->steps_since_prune += 1;
            if (mode == B2MD_PRUNE_OUTER) r->outer_steps_total += 1;
        }
        r->after_integrate = false;
    }
    if (fuse) {
        // the launch advanced the particles to the next step: its output buffer and its
        // output flag word are the inputs of the next one
        Set now = live(r);
        void *in = r->pos_cur ? r->pos_cur : now.pos_hi;
        r->pos_cur = in == now.pos_hi ? c.pos_hi_alt : now.pos_hi;
        r->gate_in = next_gate(r, r->gate_in);
        r->ahead = true;
        r->pending_kick = false;
        r->count_seen += 1;               // exactly one of this step's launches ran
    } else {
        r->ahead = false;
        r->pending_kick = true;
        // (`thermo` = this is the step the caller can observe, the last one of the call: the
        // next step is integrated by the next call)
        if (thermostatted(r) &&
            (rc = finish_thermostat_step(r, r->first_step + rep->steps_done, !thermo))) return rc;
    }
    rep->steps_done += 1;
    return 0;
}

void toggle_advance_state(b2md_runner *r) {
    Set now = live(r);
    void *in = r->pos_cur ? r->pos_cur : now.pos_hi;
    r->pos_cur = in == now.pos_hi ? r->cfg.pos_hi_alt : now.pos_hi;
    r->gate_in = next_gate(r, r->gate_in);
}

// Up to `n_inter` intermediate steps as queued one-launch steps, several per status
// read-back: a launch whose positions need a new list returns at once and makes the
// ones queued behind it return too; the device counts the launches that ran.
// Requires r->ahead.  *stop = 1 on overflow / singular.
int advance_batch(b2md_runner *r, b2md_run_report *rep, int64_t n_inter, int64_t before,
                  int *stop) {
    const b2md_runner_config &c = r->cfg;
    cudaStream_t s = r->stream;
    int rc;
    *stop = 0;
    const int m = (int)(n_inter < c.queue_depth ? n_inter : c.queue_depth);
    void *pos0 = r->pos_cur;
    const int gate0 = r->gate_in;
    for (int q = 0; q < m; ++q) {
        if ((rc = launch_advance(r))) return rc;
        toggle_advance_state(r);
    }
    if ((rc = check_cuda(cudaEventRecord(r->ev_mark, s), "mark record"))) return rc;
    if ((rc = check_cuda(cudaStreamWaitEvent(r->copy_stream, r->ev_mark, 0), "copy wait"))) return rc;
    if ((rc = check_cuda(cudaMemcpyAsync(r->h_status, c.status, sizeof(b2md_status),
                                         cudaMemcpyDeviceToHost, r->copy_stream),
                         "status read-back"))) return rc;
    if ((rc = check_cuda(cudaEventRecord(r->ev, r->copy_stream), "event record"))) return rc;
    if ((rc = check_cuda(cudaEventSynchronize(r->ev), "event sync"))) return rc;
    const int32_t *words = reinterpret_cast<const int32_t *>(r->h_status);
    const int ran = words[kWordAdvanceCount] - r->count_seen;
    r->count_seen += ran;
    // host-side state after the launches that really ran
    r->pos_cur = pos0;
    r->gate_in = gate0;
    for (int q = 0; q < ran; ++q) toggle_advance_state(r);
    rep->steps_done += ran;
    rep->max_disp2 = (double)__builtin_bit_cast(float, r->h_status->max_disp2_bits);
    r->last_disp2 = rep->max_disp2;
    if (r->h_status->singular != ~0ull) {
        if ((rc = canonicalize(r))) return rc;
        if ((rc = read_status(r))) return rc;
        rep->singular = r->h_status->singular;
        rep->reason = B2MD_RUN_SINGULAR;
        finish_report(r, rep, before);
        *stop = 1;
        return 0;
    }
    if (ran < m) {
        // the positions reached after `ran` steps need a new list
        if ((rc = canonicalize(r))) return rc;
        if ((rc = rebuild(r, rep))) return rc;
        r->gate_in = kWordRebuildFlag;
        r->last_disp2 = 0.0;
        if (!r->list_valid) {
            r->mid_step = true;
            r->ahead = false;
            rep->reason = B2MD_RUN_OVERFLOW;
            finish_report(r, rep, before);
            *stop = 1;
            return 0;
        }
    }
    return 0;
}

bool can_persist(const b2md_runner *r) {
    const b2md_runner_config &c = r->cfg;
    return c.persistent_steps > 0 && c.pair_rows == 0 && c.barrier != nullptr && can_advance(r);
}

// Up to `n_inter` intermediate steps in ONE cooperative launch (b2md_steps_persistent): the
// device loops over the steps behind grid barriers, stops before a step whose positions need
// a new list and counts the steps it took.  Requires r->ahead.  *stop = 1 on overflow /
// singular.  A launch that cannot be made (grid not co-resident) switches the mode off.
int persistent_batch(b2md_runner *r, b2md_run_report *rep, int64_t n_inter, int64_t before,
                     int *stop) {
    b2md_runner_config &c = r->cfg;
    int rc;
    *stop = 0;
    const int m = (int)(n_inter < c.persistent_steps ? n_inter : c.persistent_steps);
    Set a = live(r);
    void *in = r->pos_cur ? r->pos_cur : a.pos_hi;
    void *other = in == a.pos_hi ? c.pos_hi_alt : a.pos_hi;
    const int gate_other = r->gate_in == kWordRebuildFlag ? kWordAltFlag : kWordRebuildFlag;
    rc = b2md_steps_persistent(in, other, a.pos_lo, a.vel, a.image, c.n, &c.box, c.dt, c.ref_pos,
                               r->half_skin2, c.nbr, c.counts, c.pitch, stride_rows(r), c.boundary,
                               r->table.data(), c.ntypes, r->gate_in, gate_other, m, c.barrier,
                               c.status, r->stream);
    if (rc == -6) {                      // not co-resident on this device: per-step launches
        c.persistent_steps = 0;
        return 0;
    }
    if (rc) return rc;
    r->launches += 1;
    if ((rc = read_status(r))) return rc;
    if (r->h_status->frozen) {
        set_error("b2md_runner_run: a grid barrier of the persistent step kernel timed out");
        return -7;
    }
    const int32_t *words = reinterpret_cast<const int32_t *>(r->h_status);
    int ran = words[kWordAdvanceCount] - r->count_seen;
    if (ran < 0) ran = 0;
    if (ran > m) ran = m;
    r->count_seen += ran;
    for (int q = 0; q < ran; ++q) toggle_advance_state(r);
    rep->steps_done += ran;
    rep->max_disp2 = (double)__builtin_bit_cast(float, r->h_status->max_disp2_bits);
    r->last_disp2 = rep->max_disp2;
    if (r->h_status->singular != ~0ull) {
        if ((rc = canonicalize(r))) return rc;
        if ((rc = read_status(r))) return rc;
        rep->singular = r->h_status->singular;
        rep->reason = B2MD_RUN_SINGULAR;
        finish_report(r, rep, before);
        *stop = 1;
        return 0;
    }
    if (ran < m) {
        // the positions reached after `ran` steps need a new list
        if ((rc = canonicalize(r))) return rc;
        if ((rc = rebuild(r, rep))) return rc;
        r->gate_in = kWordRebuildFlag;
        r->last_disp2 = 0.0;
        if (!r->list_valid) {
            r->mid_step = true;
            r->ahead = false;
            rep->reason = B2MD_RUN_OVERFLOW;
            finish_report(r, rep, before);
            *stop = 1;
            return 0;
        }
    }
    return 0;
}

// A batch of graphed steps.  *stop = 1 on overflow / singular.
int graph_batch(b2md_runner *r, b2md_run_report *rep, int64_t n_batch, int64_t before, int *stop) {
    const b2md_runner_config &c = r->cfg;
    cudaStream_t s = r->stream;
    int rc;
    *stop = 0;
    if (!r->graph_exec[0] && (rc = build_graph(r, 0, 1))) return rc;
    if (r->steps_per_graph > 1 && !r->graph_exec[1] &&
        (rc = build_graph(r, 1, r->steps_per_graph))) return rc;
    k_graph_batch_reset<<<1, 1, 0, s>>>(c.status);
    int64_t left = n_batch;
    while (left > 0) {
        const bool big = r->steps_per_graph > 1 && left >= r->steps_per_graph;
        if ((rc = check_cuda(cudaGraphLaunch(r->graph_exec[big ? 1 : 0], s), "cudaGraphLaunch")))
            return rc;
        left -= big ? r->steps_per_graph : 1;
    }
    if ((rc = read_status(r))) return rc;
    const b2md_status &st = *r->h_status;
    rep->steps_done += st.graph_steps;
    rep->graph_steps += st.graph_steps;
    rep->rebuilds += st.graph_rebuilds;
    r->rebuilds_total += st.graph_rebuilds;
    if (c.reorder_mode != 0) rep->reorders += st.graph_rebuilds;
    r->launches += 1 + st.graph_steps * r->graph_launch_kernels +
                   st.graph_rebuilds * r->graph_rebuild_kernels;
    rep->max_disp2 = (double)__builtin_bit_cast(float, st.max_disp2_bits);
    if (st.graph_rebuilds) {
        rep->max_count = st.max_count;
        rep->n_boundary = st.n_boundary;
    }
    if (st.frozen) {
        // the step after the last completed one integrated, then its build overflowed
        r->list_valid = false;
        r->mid_step = true;
        r->pending_kick = false;
        rep->reason = B2MD_RUN_OVERFLOW;
        finish_report(r, rep, before);
        *stop = 1;
        return 0;
    }
    r->pending_kick = true;
    if (st.singular != ~0ull) {
        rep->singular = st.singular;
        rep->reason = B2MD_RUN_SINGULAR;
        finish_report(r, rep, before);
        *stop = 1;
    }
    return 0;
}

}  // namespace

B2MD_EXPORT void b2md_runner_destroy(b2md_runner *r);

B2MD_EXPORT b2md_runner *b2md_runner_create(const b2md_runner_config *cfg) {
    if (!cfg || cfg->n <= 0 || cfg->capacity < cfg->n || !cfg->status || !cfg->nbr ||
        cfg->ntypes < 1 || !cfg->table || cfg->stride < 1 || cfg->pitch < cfg->n ||
        !(cfg->dt > 0.0) || !(cfg->r_cut > 0.0) || cfg->skin < 0.0) {
        set_error("b2md_runner_create: bad configuration");
        return nullptr;
    }
    if (cfg->pair_rows != 0 &&
        (!cfg->pair_nbr || !cfg->pair_counts || cfg->pair_rows % 4 != 0 ||
         cfg->pair_rows < 2 * ((cfg->stride + 15) / 16 * 16) || cfg->pair_pitch % 32 != 0 ||
         cfg->pair_pitch < (cfg->n + 1) / 2)) {
        set_error("b2md_runner_create: bad pair-row buffers");
        return nullptr;
    }
    if (cfg->reorder_mode != 0 && (!cfg->keys || !cfg->keys_tmp || !cfg->perm || !cfg->perm_tmp ||
                                   !cfg->sort_scratch || cfg->reorder_every < 1 ||
                                   !cfg->pos_hi[1])) {
        set_error("b2md_runner_create: reorder buffers missing");
        return nullptr;
    }
    b2md_runner *r = new (std::nothrow) b2md_runner();
    if (!r) { set_error("b2md_runner_create: out of memory"); return nullptr; }
    r->cfg = *cfg;
    r->table.assign(cfg->table, cfg->table + 4 * cfg->ntypes * cfg->ntypes);
    r->cfg.table = r->table.data();
    r->r_list = cfg->r_cut + cfg->skin;
    r->half_skin2 = (0.5 * cfg->skin) * (0.5 * cfg->skin);
    r->current = cfg->current;
    r->pending_kick = false;
    r->list_valid = false;
    r->mid_step = false;
    r->rebuilds_total = 0;
    r->launches = 0;
    r->last_disp2 = 0.0;
    r->graph[0] = r->graph[1] = nullptr;
    r->graph_exec[0] = r->graph_exec[1] = nullptr;
    r->rebuild_exec[0] = r->rebuild_exec[1] = nullptr;
    r->rebuild_exec_kernels[0] = r->rebuild_exec_kernels[1] = 0;
    r->rebuild_seen[0] = r->rebuild_seen[1] = 0;
    r->steps_per_graph = cfg->use_graph > 1 ? cfg->use_graph : 1;
    r->pos_cur = nullptr;
    r->ahead = false;
    r->gate_in = kWordRebuildFlag;
    r->count_seen = 0;
    if (r->cfg.queue_depth < 1) r->cfg.queue_depth = 1;
    r->defer_vel = false;
    r->vel_waited = cfg->vel_ready_event == nullptr;
    r->prune_on = cfg->prune_delta > 0.0 && cfg->prune_delta < cfg->skin &&
                  0.5 * (cfg->skin - cfg->prune_delta) <= 0.125 && cfg->pair_rows > 0 &&
                  cfg->pair_nbr_inner && cfg->pair_counts_inner && cfg->pos_hi_alt &&
                  cfg->use_graph == 0 && r->cfg.queue_depth == 1;
    r->inner_state = kInnerNeedPrune;
    r->after_integrate = false;
    r->steps_since_prune = 0;
    r->refreshed = false;
    r->prunes_total = r->outer_steps_total = 0;
    r->own_h_status = r->own_stream = r->own_copy_stream = true;
    r->thermo_p = 0.0;
    r->thermo_t = 1.0;
    r->thermo_seed = 0;
    r->first_step = 0;
    r->ev_run[0] = r->ev_run[1] = nullptr;
    r->rebuild_events_used = 0;
    r->h_status = nullptr;
    r->ev = r->ev_in = r->ev_mark = nullptr;
    r->copy_stream = nullptr;
    r->stream = nullptr;
    // in-graph rebuilds always reorder (the decision cannot depend on a host counter)
    if (r->cfg.use_graph && r->cfg.reorder_mode != 0 && r->cfg.reorder_every != 1)
        r->cfg.use_graph = 0;
    if (b2md_grid_shape(&cfg->box, r->r_list, &r->grid)) { delete r; return nullptr; }
    r->own_h_status = cfg->h_status == nullptr;
    r->own_stream = cfg->run_stream == nullptr;
    r->own_copy_stream = cfg->copy_stream == nullptr;
    if (!r->own_h_status) r->h_status = static_cast<b2md_status *>(cfg->h_status);
    if (!r->own_stream) r->stream = as_stream(cfg->run_stream);
    if (!r->own_copy_stream) r->copy_stream = as_stream(cfg->copy_stream);
    if ((r->own_h_status &&
         check_cuda(cudaMallocHost((void **)&r->h_status, sizeof(b2md_status)), "cudaMallocHost")) ||
        check_cuda(cudaEventCreateWithFlags(&r->ev, cudaEventDisableTiming), "cudaEventCreate") ||
        check_cuda(cudaEventCreateWithFlags(&r->ev_in, cudaEventDisableTiming), "cudaEventCreate") ||
        check_cuda(cudaEventCreateWithFlags(&r->ev_mark, cudaEventDisableTiming), "cudaEventCreate") ||
        check_cuda(cudaEventCreate(&r->ev_run[0]), "cudaEventCreate") ||
        check_cuda(cudaEventCreate(&r->ev_run[1]), "cudaEventCreate") ||
        (r->own_copy_stream &&
         check_cuda(cudaStreamCreateWithFlags(&r->copy_stream, cudaStreamNonBlocking),
                    "cudaStreamCreate")) ||
        (r->own_stream &&
         check_cuda(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking),
                    "cudaStreamCreate"))) {
        b2md_runner_destroy(r);
        return nullptr;
    }
    return r;
}

B2MD_EXPORT void b2md_runner_destroy(b2md_runner *r) {
    if (!r) return;
    destroy_graph(r);
    if (r->h_status && r->own_h_status) cudaFreeHost(r->h_status);
    if (r->ev) cudaEventDestroy(r->ev);
    if (r->ev_in) cudaEventDestroy(r->ev_in);
    if (r->ev_mark) cudaEventDestroy(r->ev_mark);
    for (cudaEvent_t e : r->ev_run) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : r->ev_rebuild) if (e) cudaEventDestroy(e);
    // lent streams may still carry this runner's work: drain before the events go
    if (r->stream && !r->own_stream) cudaStreamSynchronize(r->stream);
    if (r->copy_stream && !r->own_copy_stream) cudaStreamSynchronize(r->copy_stream);
    if (r->copy_stream && r->own_copy_stream) cudaStreamDestroy(r->copy_stream);
    if (r->stream && r->own_stream) cudaStreamDestroy(r->stream);
    delete r;
}

B2MD_EXPORT int b2md_runner_set_list(b2md_runner *r, int32_t *nbr, int32_t stride) {
    if (!r || !nbr || stride < 1) { set_error("b2md_runner_set_list: bad arguments"); return -1; }
    r->cfg.nbr = nbr;
    r->cfg.stride = stride;
    r->list_valid = false;
    destroy_graph(r);          // the list pointer and stride are baked into the graph
    return 0;
}

B2MD_EXPORT int b2md_runner_set_pair_list(b2md_runner *r, int32_t *pair_nbr, int32_t pair_rows) {
    if (!r || !pair_nbr || pair_rows % 4 != 0 || pair_rows < 2 * stride_rows(r)) {
        set_error("b2md_runner_set_pair_list: bad arguments");
        return -1;
    }
    r->cfg.pair_nbr = pair_nbr;
    r->cfg.pair_rows = pair_rows;
    r->list_valid = false;
    destroy_graph(r);
    return 0;
}

B2MD_EXPORT int b2md_runner_set_inner_pair_list(b2md_runner *r, int32_t *pair_nbr_inner) {
    if (!r || (r->prune_on && !pair_nbr_inner)) {
        set_error("b2md_runner_set_inner_pair_list: bad arguments");
        return -1;
    }
    r->cfg.pair_nbr_inner = pair_nbr_inner;
    r->inner_state = kInnerNeedPrune;
    r->list_valid = false;
    return 0;
}

B2MD_EXPORT int64_t b2md_runner_prune_count(const b2md_runner *r, int64_t *outer_steps) {
    if (!r) return -1;
    if (outer_steps) *outer_steps = r->outer_steps_total;
    return r->prunes_total;
}

B2MD_EXPORT int b2md_runner_set_thermostat(b2md_runner *r, double probability,
                                           double temperature, uint64_t seed) {
    if (!r || !(probability >= 0.0) || !(temperature > 0.0)) {
        set_error("b2md_runner_set_thermostat: bad arguments");
        return -1;
    }
    if (probability > 0.0 && (r->pending_kick || r->ahead)) {
        set_error("b2md_runner_set_thermostat: a half-kick is pending; finish the run first");
        return -2;
    }
    r->thermo_p = probability > 1.0 ? 1.0 : probability;
    r->thermo_t = temperature;
    r->thermo_seed = seed;
    if (probability > 0.0) {
        // fused half-kicks and captured steps have no slot for the thermostat
        r->cfg.use_graph = 0;
        destroy_graph(r);
    }
    return 0;
}

B2MD_EXPORT int b2md_runner_set_step(b2md_runner *r, int64_t first_step) {
    if (!r || first_step < 0) { set_error("b2md_runner_set_step: bad arguments"); return -1; }
    r->first_step = first_step;
    return 0;
}

B2MD_EXPORT int b2md_runner_prepare(b2md_runner *r, b2md_run_report *rep) {
    if (!r || !rep) { set_error("b2md_runner_prepare: null argument"); return -1; }
    *rep = b2md_run_report();
    const int64_t before = r->launches;
    int rc = order_after_caller(r);
    if (rc) return rc;
    if ((rc = begin_call(r))) return rc;
    r->defer_vel = !r->vel_waited && r->cfg.use_graph == 0;
    if ((rc = rebuild(r, rep))) return rc;
    if (!r->vel_waited) {
        // (a path that did not gather: graph mode keeps the row order inside this call)
        if ((rc = check_cuda(cudaStreamWaitEvent(r->stream,
                                                 static_cast<cudaEvent_t>(r->cfg.vel_ready_event), 0),
                             "velocity upload wait"))) return rc;
        r->defer_vel = false;
        r->vel_waited = true;
    }
    if (!r->list_valid) {
        rep->reason = B2MD_RUN_OVERFLOW;
        finish_report(r, rep, before);
        return 0;
    }
    if ((rc = launch_force(r, true))) return rc;
    if ((rc = read_status(r))) return rc;
    r->mid_step = false;
    rep->singular = r->h_status->singular;
    rep->reason = r->h_status->singular != ~0ull ? B2MD_RUN_SINGULAR : B2MD_RUN_DONE;
    finish_report(r, rep, before);
    return 0;
}

B2MD_EXPORT int b2md_runner_run(b2md_runner *r, int64_t n_steps, int32_t finalize_at_end,
                                b2md_run_report *rep) {
    if (!r || !rep || n_steps < 0) { set_error("b2md_runner_run: bad arguments"); return -1; }
    *rep = b2md_run_report();
    const int64_t before = r->launches;
    const b2md_runner_config &c = r->cfg;
    int rc, stop = 0;
    if (!r->list_valid && !r->mid_step) {
        set_error("b2md_runner_run: no valid neighbour list; call b2md_runner_prepare first");
        return -2;
    }
    if ((rc = order_after_caller(r))) return rc;
    if ((rc = begin_call(r))) return rc;
    // The advance counter lives in the status block the public operators share and reset
    // (b2md_status_reset): start every call from a known value instead of trusting the
    // host mirror across calls.
    if ((rc = check_cuda(cudaMemsetAsync(reinterpret_cast<int32_t *>(c.status) + kWordAdvanceCount,
                                         0, sizeof(int32_t), r->stream), "counter reset")))
        return rc;
    r->count_seen = 0;
    if (r->mid_step) {
        // previous call stopped on overflow after integrating: finish that step
        if ((rc = rebuild(r, rep))) return rc;
        if (!r->list_valid) {
            rep->reason = B2MD_RUN_OVERFLOW;
            finish_report(r, rep, before);
            return 0;
        }
        if ((rc = launch_force(r, rep->steps_done + 1 >= n_steps))) return rc;
        r->mid_step = false;
        r->pending_kick = true;
        if (thermostatted(r) && (rc = finish_thermostat_step(r, r->first_step + rep->steps_done)))
            return rc;
        rep->steps_done += 1;
    }
    while (rep->steps_done < n_steps) {
        const int64_t left = n_steps - rep->steps_done;
        // graphed steps need the fused kick and must not be the observable last step
        if (c.use_graph && r->pending_kick && left > 1) {
            if ((rc = graph_batch(r, rep, left - 1, before, &stop))) return rc;
        } else if (r->ahead && left > 1 && can_persist(r)) {
            if ((rc = persistent_batch(r, rep, left - 1, before, &stop))) return rc;
        } else if (c.queue_depth > 1 && r->ahead && left > 1 && can_advance(r)) {
            if ((rc = advance_batch(r, rep, left - 1, before, &stop))) return rc;
        } else {
            // energies / virial only on the step the caller can observe (the last one)
            if ((rc = plain_step(r, rep, left == 1, before, &stop))) return rc;
        }
        if (stop) return 0;
    }
    if (finalize_at_end && r->pending_kick) {
        Set a = live(r);
        if ((rc = b2md_vv_finalize(a.vel, a.force, c.n, c.dt, r->stream))) return rc;
        r->launches += 1;
        r->pending_kick = false;
    }
    if ((rc = read_status(r))) return rc;   // also drains the stream
    rep->singular = r->h_status->singular;
    rep->reason = r->h_status->singular != ~0ull ? B2MD_RUN_SINGULAR : B2MD_RUN_DONE;
    finish_report(r, rep, before);
    return 0;
}

// ---- native loop of the all-to-all force mode ------------------------------------
// Simulation.run with force_mode = "all_to_all" (the reference's default, sim.py:62-102):
// integrate -> compute_forces_all_to_all -> finalize [-> thermostat] per step.  No list, no
// rebuild flag, nothing the host has to look at between steps: the whole call is enqueued
// without a round trip and the status block -- the singular-pair word -- is read once per chunk
// of kAllPairsChunk steps.  With a second buffer for the position high words an intermediate
// step is ONE launch (b2md_force_lj_all_pairs_advance: force + finalize + integrate of the next
// step by the thread that holds the particle's total force); without it finalize of step s and
// integrate of step s + 1 share one pass over the state; a thermostatted step is the force
// kernel plus b2md_vv_finalize_andersen.  Same operations in the same order as the operator
// loop: bit-identical trajectories.
constexpr int64_t kAllPairsChunk = 512;

B2MD_EXPORT int b2md_run_all_pairs(void *d_pos_hi, void *d_pos_lo, void *d_vel, void *d_force_f4,
                                   void *d_image_i4, float *d_virial, int64_t n,
                                   const b2md_box *box, const double *table, int32_t ntypes,
                                   double dt, int64_t n_steps, double thermo_probability,
                                   double thermo_temperature, uint64_t thermo_seed,
                                   int64_t first_step, void *d_pos_hi_alt, b2md_status *d_status,
                                   void *h_status, void *stream, b2md_run_report *rep) {
    if (!d_pos_hi || !d_pos_lo || !d_vel || !d_force_f4 || !d_image_i4 || !box || !table ||
        !d_status || !h_status || !rep || n < 1 || n_steps < 0 || !(thermo_probability >= 0.0)) {
        set_error("b2md_run_all_pairs: bad arguments");
        return -1;
    }
    *rep = b2md_run_report();
    cudaStream_t s = as_stream(stream);
    const bool thermostatted = thermo_probability > 0.0;
    const double p = thermo_probability > 1.0 ? 1.0 : thermo_probability;
    b2md_status *h = static_cast<b2md_status *>(h_status);
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int rc;
    if ((rc = check_cuda(cudaEventCreate(&ev[0]), "event create"))) return rc;
    if ((rc = check_cuda(cudaEventCreate(&ev[1]), "event create"))) {
        cudaEventDestroy(ev[0]);
        return rc;
    }
    auto leave = [&](int code) {
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        return code;
    };
    if ((rc = b2md_status_reset(d_status, stream))) return leave(rc);
    if ((rc = check_cuda(cudaEventRecord(ev[0], s), "event record"))) return leave(rc);
    bool pending_kick = false;          // forces of the last step not yet applied to the velocities
    bool ahead = false;                 // the next step is already integrated
    // One launch per intermediate step (b2md_force_lj_all_pairs_advance) when the caller lends
    // a second buffer for the position high words: they ping-pong between the two.
    const bool fuse = d_pos_hi_alt != nullptr && d_pos_hi_alt != d_pos_hi && !thermostatted;
    void *cur = d_pos_hi, *other = d_pos_hi_alt;
    while (rep->steps_done < n_steps) {
        const int64_t chunk = std::min<int64_t>(kAllPairsChunk, n_steps - rep->steps_done);
        for (int64_t q = 0; q < chunk; ++q) {
            if (!ahead) {
                if (pending_kick)
                    rc = b2md_vv_finalize_integrate(cur, d_pos_lo, d_vel, d_force_f4,
                                                    d_image_i4, n, box, dt, nullptr, 0.0, d_status,
                                                    stream);
                else
                    rc = b2md_vv_integrate(cur, d_pos_lo, d_vel, d_force_f4, d_image_i4, n,
                                           box, dt, nullptr, 0.0, d_status, stream);
                if (rc) return leave(rc);
                rep->kernel_launches += 1;
            }
            ahead = false;
            if (fuse && rep->steps_done + q + 1 < n_steps) {
                // force(s) + finalize(s) + integrate(s + 1) in one launch
                if ((rc = b2md_force_lj_all_pairs_advance(cur, other, d_pos_lo, d_vel, d_image_i4, n,
                                                          box, table, ntypes, dt, d_status, stream)))
                    return leave(rc);
                rep->kernel_launches += 1;
                std::swap(cur, other);
                ahead = true;
                pending_kick = false;
                continue;
            }
            if ((rc = b2md_force_lj_all_pairs(cur, n, box, table, ntypes, d_force_f4, d_virial,
                                              d_status, stream))) return leave(rc);
            rep->kernel_launches += 1;
            pending_kick = true;
            if (thermostatted) {
                // finalize + thermostat (+ integrate of the next step unless this is the
                // step the caller observes) in one pass
                const bool more = rep->steps_done + q + 1 < n_steps;
                if ((rc = b2md_vv_finalize_andersen(d_pos_hi, d_pos_lo, d_vel, d_force_f4,
                                                    d_image_i4, n, box, dt, thermo_seed,
                                                    (uint64_t)(first_step + rep->steps_done + q),
                                                    p, thermo_temperature, more ? 1 : 0, nullptr,
                                                    0.0, d_status, stream))) return leave(rc);
                rep->kernel_launches += 1;
                pending_kick = false;
                ahead = more;
            }
        }
        rep->steps_done += chunk;
        const bool last = rep->steps_done >= n_steps;
        if (last && pending_kick) {
            if ((rc = b2md_vv_finalize(d_vel, d_force_f4, n, dt, stream))) return leave(rc);
            rep->kernel_launches += 1;
            pending_kick = false;
        }
        if (last && cur != d_pos_hi) {
            if ((rc = check_cuda(cudaMemcpyAsync(d_pos_hi, cur, (size_t)n * 4 * sizeof(float),
                                                 cudaMemcpyDeviceToDevice, s), "position copy")))
                return leave(rc);
            std::swap(cur, other);
        }
        if (last && (rc = check_cuda(cudaEventRecord(ev[1], s), "event record"))) return leave(rc);
        if ((rc = check_cuda(cudaMemcpyAsync(h, d_status, sizeof(b2md_status),
                                             cudaMemcpyDeviceToHost, s), "status read-back")))
            return leave(rc);
        if ((rc = check_cuda(cudaStreamSynchronize(s), "status sync"))) return leave(rc);
        if (h->singular != ~0ull) {
            // a coincident pair (forces.py:113-116): the steps enqueued behind it ran on
            // non-finite forces; stop here and let the caller raise
            if (pending_kick) {
                if ((rc = b2md_vv_finalize(d_vel, d_force_f4, n, dt, stream))) return leave(rc);
                rep->kernel_launches += 1;
            }
            if (cur != d_pos_hi &&
                (rc = check_cuda(cudaMemcpyAsync(d_pos_hi, cur, (size_t)n * 4 * sizeof(float),
                                                 cudaMemcpyDeviceToDevice, s), "position copy")))
                return leave(rc);
            if (!last && (rc = check_cuda(cudaEventRecord(ev[1], s), "event record")))
                return leave(rc);
            if ((rc = check_cuda(cudaStreamSynchronize(s), "drain"))) return leave(rc);
            break;
        }
    }
    if (n_steps == 0) {
        if ((rc = check_cuda(cudaEventRecord(ev[1], s), "event record"))) return leave(rc);
        if ((rc = check_cuda(cudaMemcpyAsync(h, d_status, sizeof(b2md_status),
                                             cudaMemcpyDeviceToHost, s), "status read-back")))
            return leave(rc);
        if ((rc = check_cuda(cudaStreamSynchronize(s), "status sync"))) return leave(rc);
    }
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, ev[0], ev[1]) == cudaSuccess) rep->gpu_ms = ms;
    rep->singular = h->singular;
    rep->reason = h->singular != ~0ull ? B2MD_RUN_SINGULAR : B2MD_RUN_DONE;
    rep->list_valid = 1;
    return leave(0);
}
