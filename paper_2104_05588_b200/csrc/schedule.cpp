// Host schedule of DASO: warm-up / cycling / cool-down phases and the B,S
// halving / reset rule (§3), with the readings R6, R8-R10, R13-R15
// of DESIGN.md §3.  Bit-exact contract with the independent CPU oracle
// (oracle/schedule.py), checked record by record in tests/test_schedule_abi.py.
#include <cmath>
#include <new>

#include "daso_internal.h"

namespace daso {

int resolved_S(const daso_sched_config& c) {
    return c.S_init < 0 ? std::max(1, c.B_init / 4) : c.S_init;   // P:99 "initial value of B/4"
}

const char* validate_sched(const daso_sched_config& c) {
    int S = resolved_S(c);
    if (c.B_init < 1) return "B must be >= 1";
    if (c.gpus_per_node < 1) return "gpus_per_node must be >= 1";
    if (S < 0 || S > c.B_init) return "S must satisfy 0 <= S <= B";
    if (c.total_epochs < 1) return "total_epochs must be >= 1";
    if (c.steps_per_epoch < 1) return "steps_per_epoch must be >= 1";
    if (c.warmup_epochs < 0 || c.cooldown_epochs < 0 ||
        (int64_t)c.warmup_epochs + c.cooldown_epochs > c.total_epochs)
        return "warmup_epochs + cooldown_epochs must be <= total_epochs";
    for (int b = c.B_init;; b = std::max(1, b / 2)) {   // every B of the halving chain divides an epoch (R10)
        if (c.steps_per_epoch % b != 0) return "every B of the halving chain must divide steps_per_epoch";
        if (b == 1) break;
    }
    return nullptr;
}

int phase_of(int64_t epoch, const daso_sched_config& c) {
    if (epoch < c.warmup_epochs) return DASO_WARMUP;
    if (epoch >= (int64_t)c.total_epochs - c.cooldown_epochs) return DASO_COOLDOWN;
    return DASO_CYCLING;
}

Schedule::Schedule(const daso_sched_config& c) : cfg(c) {
    B = c.B_init;
    S = resolved_S(c);
}

daso_record Schedule::next(int plateau) {
    const int64_t k = step;
    const int64_t spe = cfg.steps_per_epoch;
    const int64_t e = k / spe;
    int64_t action = 0;
    if (k % spe == 0) {
        if (k > 0 && plateau == 1 && phase_of(e - 1, cfg) == DASO_CYCLING) {
            if (B > 1 || S > 1) {              // P:99 "reduced by a factor of two, down to a minimum of one"
                B = std::max(1, B / 2);
                S = (S == 0) ? 0 : std::max(1, S / 2);
                action = 1;
            } else {                           // P:99 "When B, W = 1 ... reset to their initial values"
                B = cfg.B_init;
                S = resolved_S(cfg);
                action = 2;
            }
        }
        batch_in_cycle = 0;                    // cycles restart every epoch (R10)
    }
    const int ph = phase_of(e, cfg);

    daso_record r{};
    r.merge_group = -1;
    r.merge_sent = -1;
    if (has_pending && pend_due == k) {        // due merge before any new send (R6, R8)
        r.merge = 1;
        r.merge_S = pend_S;
        r.merge_group = pend_group;
        r.merge_sent = pend_sent;
        has_pending = false;
    }
    int64_t bic = 0, send = 0, blocking = 0;
    if (ph == DASO_CYCLING) {
        bic = batch_in_cycle;
        send = (bic == 0);                     // "every B-th batch", first cycling batch sends (R15)
        blocking = (send && S == 0);
        batch_in_cycle = (int)((bic + 1) % B);
    } else {
        send = 1;                              // P:86 blocking: "all synchronization steps ... after each batch"
        blocking = 1;
    }
    int64_t group = -1;
    if (send) {
        group = n_syncs % cfg.gpus_per_node;   // rotation, R9
        n_syncs += 1;
        if (!blocking) {
            has_pending = true;
            pend_due = k + S;
            pend_S = S;
            pend_group = (int)group;
            pend_sent = k;
        }
    }
    r.step = k;
    r.epoch = e;
    r.phase = ph;
    r.B = B;
    r.S = S;
    r.batch_in_cycle = bic;
    r.plateau_action = action;
    r.send = send;
    r.blocking = blocking;
    r.send_group = group;
    r.n_syncs = n_syncs;
    r.pending = has_pending ? 1 : 0;
    r.due = has_pending ? pend_due : -1;
    step += 1;
    return r;
}

// Loss-plateau detector ("not decreasing by more than a set percentage threshold",
// P:172 "stable for 5 epochs"; reading R20): an epoch improves iff
// loss < best - threshold * |best|; `patience` consecutive non-improving epochs fire.
struct Plateau {
    int patience;
    double threshold;
    double best = INFINITY;
    int stable = 0;
    int update(double loss) {
        if (std::isinf(best) || loss < best - threshold * std::fabs(best)) {
            best = loss;
            stable = 0;
            return 0;
        }
        if (++stable >= patience) {
            stable = 0;
            return 1;
        }
        return 0;
    }
};

}  // namespace daso

extern "C" {

daso_status daso_plateau_create(int patience, double threshold, daso_plateau** out) {
    if (!out) return DASO_ERR_ARGUMENT;
    if (patience < 1 || !(threshold >= 0)) return DASO_ERR_CONFIG;
    auto* p = new (std::nothrow) daso::Plateau{patience, threshold};
    if (!p) return DASO_ERR_ARGUMENT;
    *out = reinterpret_cast<daso_plateau*>(p);
    return DASO_OK;
}

daso_status daso_plateau_update(daso_plateau* h, double loss, int* fired) {
    if (!h || !fired) return DASO_ERR_ARGUMENT;
    if (!std::isfinite(loss)) return DASO_ERR_NONFINITE;
    *fired = reinterpret_cast<daso::Plateau*>(h)->update(loss);
    return DASO_OK;
}

daso_status daso_plateau_destroy(daso_plateau* h) {
    delete reinterpret_cast<daso::Plateau*>(h);
    return DASO_OK;
}

daso_status daso_lr_at(int64_t step, int steps_per_epoch, double base_lr, int world, int warmup_epochs,
                       double factor, int n_plateaus, double* out) {
    if (!out) return DASO_ERR_ARGUMENT;
    if (steps_per_epoch < 1 || world < 1 || warmup_epochs < 0 || step < 0 || n_plateaus < 0) return DASO_ERR_CONFIG;
    const double peak = base_lr * world;                       // P:172 "scaled with the number of global processes"
    const int64_t warm = int64_t(warmup_epochs) * steps_per_epoch;
    if (step < warm) {
        *out = peak * double(step + 1) / double(warm);          // P:212 "increased from 0.0 to" the peak
    } else {
        *out = peak * std::pow(factor, double(n_plateaus));    // P:162 "decreases the learning rate by a set factor"
    }
    return DASO_OK;
}

daso_status daso_sched_create(const daso_sched_config* cfg, daso_sched** out) {
    if (!cfg || !out) return DASO_ERR_ARGUMENT;
    if (daso::validate_sched(*cfg)) return DASO_ERR_CONFIG;
    try {
        *out = reinterpret_cast<daso_sched*>(new daso::Schedule(*cfg));
    } catch (...) {
        return DASO_ERR_ARGUMENT;
    }
    return DASO_OK;
}

daso_status daso_sched_next(daso_sched* s, int plateau, daso_record* out) {
    if (!s || !out) return DASO_ERR_ARGUMENT;
    *out = reinterpret_cast<daso::Schedule*>(s)->next(plateau);
    return DASO_OK;
}

daso_status daso_sched_destroy(daso_sched* s) {
    delete reinterpret_cast<daso::Schedule*>(s);
    return DASO_OK;
}

}  // extern "C"
