// Native step loop: Simulation.run / SignalEngine.run_steps (reference
// core.py:262-279) with the rebuild policy of Simulation._compute_forces and
// _rebuild (sim.py:114-149), driven from C++.
//
// Per MD step the stream sees
//     k_integrate<2>   finalize(s-1) + integrate(s) + displacement check
//     64-byte D2H      status block -> pinned host copy, then an event
//     k_force_lj       launched speculatively with the current list
// and the host inspects the rebuild flag while the force kernel is running.  In
// the common case (flag clear) nothing else happens and the GPU never idles.  If
// the flag is set, the speculative forces are discarded: bin -> optional reorder
// -> list build -> snapshot, the overflow word is read (one sync per rebuild),
// and the force kernel is launched again on the fresh list.
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
    cudaEvent_t ev;
    int64_t launches;
};

namespace {

struct Set {
    void *pos_hi, *pos_lo, *vel, *force, *image;
    float *virial;
};

Set live(const b2md_runner *r) {
    const b2md_runner_config &c = r->cfg;
    const int k = r->current;
    return Set{c.pos_hi[k], c.pos_lo[k], c.vel[k], c.force[k], c.image[k], c.virial[k]};
}

Set spare(const b2md_runner *r) {
    const b2md_runner_config &c = r->cfg;
    const int k = 1 - r->current;
    return Set{c.pos_hi[k], c.pos_lo[k], c.vel[k], c.force[k], c.image[k], c.virial[k]};
}

int read_status(b2md_runner *r) {
    cudaStream_t s = as_stream(r->cfg.stream);
    int rc = check_cuda(cudaMemcpyAsync(r->h_status, r->cfg.status, sizeof(b2md_status),
                                        cudaMemcpyDeviceToHost, s), "status read-back");
    if (rc) return rc;
    return check_cuda(cudaStreamSynchronize(s), "status sync");
}

// thermo = false on steps whose per-particle energies cannot be observed
int launch_force(b2md_runner *r, bool thermo) {
    const b2md_runner_config &c = r->cfg;
    Set a = live(r);
    r->launches += 1;
    return b2md_force_lj(a.pos_hi, c.n, &c.box, c.nbr, c.counts, c.pitch, (c.stride + 15) / 16 * 16,
                         c.boundary, r->table.data(), c.ntypes,
                         thermo ? 0 : B2MD_FORCE_SKIP_THERMO, a.force, a.virial, c.status,
                         c.stream);
}

int reorder(b2md_runner *r) {
    const b2md_runner_config &c = r->cfg;
    Set a = live(r), b = spare(r);
    int rc;
    int key_bits;
    if (c.reorder_mode == 1) {
        rc = b2md_hilbert_keys(a.pos_hi, a.pos_lo, c.n, &r->grid, c.hilbert_bits, c.keys, c.stream);
        key_bits = b2md_hilbert_key_bits(&r->grid, c.hilbert_bits);
        if (key_bits < 0) { set_error("reorder: Hilbert key does not fit"); return -5; }
    } else {
        // cell order needs the cell of every particle first
        rc = b2md_bin(a.pos_hi, a.pos_lo, c.n, &r->grid, c.cell_of, c.cell_start,
                      c.cell_particles, c.bin_scratch, c.stream);
        r->launches += 6;
        if (rc) return rc;
        rc = b2md_cell_keys(c.cell_of, c.n, c.keys, c.stream);
        key_bits = 1;
        while ((1ll << key_bits) < r->grid.n_cells) ++key_bits;
    }
    if (rc) return rc;
    if ((rc = b2md_iota_i32(c.perm, c.n, c.stream))) return rc;
    if ((rc = b2md_sort_pairs_u64(c.keys, c.perm, c.keys_tmp, c.perm_tmp, c.n, key_bits,
                                  c.sort_scratch, c.stream))) return rc;
    r->launches += 2 + 5 * ((key_bits + 7) / 8);
    if ((rc = b2md_gather16(a.pos_hi, b.pos_hi, c.perm, c.n, c.stream))) return rc;
    if ((rc = b2md_gather16(a.pos_lo, b.pos_lo, c.perm, c.n, c.stream))) return rc;
    if ((rc = b2md_gather16(a.vel, b.vel, c.perm, c.n, c.stream))) return rc;
    if ((rc = b2md_gather16(a.force, b.force, c.perm, c.n, c.stream))) return rc;
    if ((rc = b2md_gather16(a.image, b.image, c.perm, c.n, c.stream))) return rc;
    if ((rc = b2md_gather4(a.virial, b.virial, c.perm, c.n, c.stream))) return rc;
    r->launches += 6;
    r->current = 1 - r->current;
    return 0;
}

// bin -> (reorder) -> build -> snapshot; leaves overflow/max_count in h_status.
int rebuild(b2md_runner *r, b2md_run_report *rep) {
    const b2md_runner_config &c = r->cfg;
    int rc;
    if (c.reorder_mode != 0 && (r->rebuilds_total % c.reorder_every) == 0) {
        if ((rc = reorder(r))) return rc;
        rep->reorders += 1;
    }
    Set a = live(r);
    if ((rc = b2md_status_reset_list(c.status, c.stream))) return rc;
    if ((rc = b2md_bin(a.pos_hi, a.pos_lo, c.n, &r->grid, c.cell_of, c.cell_start,
                       c.cell_particles, c.bin_scratch, c.stream))) return rc;
    if ((rc = b2md_build_nlist(a.pos_hi, a.pos_lo, c.n, &c.box, &r->grid, c.cell_of,
                               c.cell_start, c.cell_particles, r->r_list, c.stride, c.pitch,
                               c.nbr, c.counts, c.boundary, r->r_list + c.skin, c.n,
                               c.status, c.stream))) return rc;
    if ((rc = b2md_snapshot(a.pos_hi, a.pos_lo, a.image, c.n, &c.box, c.at_build, c.ref_pos,
                            c.stream))) return rc;
    r->launches += 1 + 6 + 2 + 1;
    r->rebuilds_total += 1;
    rep->rebuilds += 1;
    if ((rc = read_status(r))) return rc;
    rep->max_count = r->h_status->max_count;
    rep->n_boundary = r->h_status->n_boundary;
    r->list_valid = r->h_status->overflow == 0;
    return 0;
}

void finish_report(b2md_runner *r, b2md_run_report *rep, int64_t launches_before) {
    rep->current = r->current;
    rep->kernel_launches = r->launches - launches_before;
    rep->list_valid = r->list_valid ? 1 : 0;
}

}  // namespace

B2MD_EXPORT b2md_runner *b2md_runner_create(const b2md_runner_config *cfg) {
    if (!cfg || cfg->n <= 0 || cfg->capacity < cfg->n || !cfg->status || !cfg->nbr ||
        cfg->ntypes < 1 || !cfg->table || cfg->stride < 1 || cfg->pitch < cfg->n ||
        !(cfg->dt > 0.0) || !(cfg->r_cut > 0.0) || cfg->skin < 0.0) {
        set_error("b2md_runner_create: bad configuration");
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
    if (b2md_grid_shape(&cfg->box, r->r_list, &r->grid)) { delete r; return nullptr; }
    if (check_cuda(cudaMallocHost((void **)&r->h_status, sizeof(b2md_status)), "cudaMallocHost") ||
        check_cuda(cudaEventCreateWithFlags(&r->ev, cudaEventDisableTiming), "cudaEventCreate")) {
        delete r;
        return nullptr;
    }
    return r;
}

B2MD_EXPORT void b2md_runner_destroy(b2md_runner *r) {
    if (!r) return;
    cudaFreeHost(r->h_status);
    cudaEventDestroy(r->ev);
    delete r;
}

B2MD_EXPORT int b2md_runner_set_list(b2md_runner *r, int32_t *nbr, int32_t stride) {
    if (!r || !nbr || stride < 1) { set_error("b2md_runner_set_list: bad arguments"); return -1; }
    r->cfg.nbr = nbr;
    r->cfg.stride = stride;
    r->list_valid = false;
    return 0;
}

B2MD_EXPORT int b2md_runner_prepare(b2md_runner *r, b2md_run_report *rep) {
    if (!r || !rep) { set_error("b2md_runner_prepare: null argument"); return -1; }
    *rep = b2md_run_report();
    const int64_t before = r->launches;
    int rc = rebuild(r, rep);
    if (rc) return rc;
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
    cudaStream_t s = as_stream(c.stream);
    int rc;
    if (!r->list_valid && !r->mid_step) {
        set_error("b2md_runner_run: no valid neighbour list; call b2md_runner_prepare first");
        return -2;
    }
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
        rep->steps_done += 1;
    }
    while (rep->steps_done < n_steps) {
        Set a = live(r);
        if (r->pending_kick)
            rc = b2md_vv_finalize_integrate(a.pos_hi, a.pos_lo, a.vel, a.force, a.image, c.n,
                                            &c.box, c.dt, c.ref_pos, r->half_skin2, c.status, s);
        else
            rc = b2md_vv_integrate(a.pos_hi, a.pos_lo, a.vel, a.force, a.image, c.n, &c.box, c.dt,
                                   c.ref_pos, r->half_skin2, c.status, s);
        if (rc) return rc;
        r->launches += 1;
        r->pending_kick = false;
        if ((rc = check_cuda(cudaMemcpyAsync(r->h_status, c.status, sizeof(b2md_status),
                                             cudaMemcpyDeviceToHost, s), "flag read-back")))
            return rc;
        if ((rc = check_cuda(cudaEventRecord(r->ev, s), "event record"))) return rc;
        // energies / virial only on the step the caller can observe (the last one)
        const bool thermo = rep->steps_done + 1 >= n_steps;
        if ((rc = launch_force(r, thermo))) return rc;     // speculative
        if ((rc = check_cuda(cudaEventSynchronize(r->ev), "event sync"))) return rc;
        rep->max_disp2 = (double)__builtin_bit_cast(float, r->h_status->max_disp2_bits);
        if (r->h_status->singular != ~0ull) {
            // a force evaluation of an earlier step met a coincident pair
            // (forces.py:113-116); stop after draining the stream
            if ((rc = read_status(r))) return rc;
            rep->singular = r->h_status->singular;
            rep->reason = B2MD_RUN_SINGULAR;
            r->pending_kick = true;
            rep->steps_done += 1;
            finish_report(r, rep, before);
            return 0;
        }
        if (r->h_status->rebuild_flag) {
            rep->wasted_force_launches += 1;
            if ((rc = rebuild(r, rep))) return rc;
            if (!r->list_valid) {
                r->mid_step = true;
                rep->reason = B2MD_RUN_OVERFLOW;
                finish_report(r, rep, before);
                return 0;
            }
            if ((rc = launch_force(r, thermo))) return rc;
        }
        r->pending_kick = true;
        rep->steps_done += 1;
    }
    if (finalize_at_end && r->pending_kick) {
        Set a = live(r);
        if ((rc = b2md_vv_finalize(a.vel, a.force, c.n, c.dt, s))) return rc;
        r->launches += 1;
        r->pending_kick = false;
    }
    if ((rc = read_status(r))) return rc;   // also drains the stream
    rep->singular = r->h_status->singular;
    rep->reason = r->h_status->singular != ~0ull ? B2MD_RUN_SINGULAR : B2MD_RUN_DONE;
    finish_report(r, rep, before);
    return 0;
}
