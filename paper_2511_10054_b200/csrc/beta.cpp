// Adaptive distribution-gate threshold (gating.derive_beta / BetaController,
// gating.py:173-221) as plain host functions over a caller-owned state, used
// by the decode engine and, through the C-ABI, by gating.BetaController, so
// one implementation serves both. f64 operations in the reference's order
// (each product and sum rounded on its own: no contraction).
#include <string.h>

#include "../../include/bmoe.h"

namespace bm {
void set_error(const char *fmt, ...);
}

extern "C" int bm_derive_beta(double budget_bytes, double expert_bytes, const double *grid_host,
                              const double *nhat_host, int32_t n, double current_beta, double *beta_out) {
    if (!beta_out || n < 0 || (n > 0 && (!grid_host || !nhat_host))) {
        bm::set_error("bm_derive_beta: bad arguments");
        return BM_EINVAL;
    }
    if (expert_bytes < 0.0 || budget_bytes < 0.0) {
        bm::set_error("budget and expert bytes must be nonnegative");
        return BM_EINVAL;
    }
    bool any = false;
    double best = 0.0;
    for (int32_t i = 0; i < n; ++i) {
        volatile double vol = nhat_host[i] * expert_bytes;  // estimated admitted volume at this candidate
        if (vol <= budget_bytes && (!any || grid_host[i] > best)) {
            best = grid_host[i];
            any = true;
        }
    }
    *beta_out = any ? best : current_beta;
    return BM_OK;
}

extern "C" int bm_beta_init(bm_beta_state *s, double budget_bytes, double expert_bytes, double initial_beta,
                            const double *grid_host, int32_t n, double decay, int64_t period) {
    if (!s || !grid_host || n < 1 || n > BM_BETA_MAX_GRID) {
        bm::set_error("bm_beta_init: need 1..%d grid values", BM_BETA_MAX_GRID);
        return n < 1 ? BM_ECONFIG : BM_EINVAL;
    }
    if (!(decay >= 0.0 && decay < 1.0) || period < 1) {
        bm::set_error("bm_beta_init: decay must be in [0, 1) and period >= 1");
        return BM_ECONFIG;
    }
    memset(s, 0, sizeof(*s));
    s->budget_bytes = budget_bytes;
    s->expert_bytes = expert_bytes;
    s->beta = initial_beta;
    s->decay = decay;
    s->period = period;
    s->n_grid = n;
    // the reference sorts the grid (np.asarray(sorted(grid)))
    for (int32_t i = 0; i < n; ++i) s->grid[i] = grid_host[i];
    for (int32_t i = 1; i < n; ++i)
        for (int32_t j = i; j > 0 && s->grid[j - 1] > s->grid[j]; --j) {
            const double t = s->grid[j];
            s->grid[j] = s->grid[j - 1];
            s->grid[j - 1] = t;
        }
    return BM_OK;
}

extern "C" int bm_beta_record(bm_beta_state *s, double delta, int64_t miss_count, double *beta_out) {
    if (!s) return BM_EINVAL;
    const double omd = 1.0 - s->decay;
    for (int32_t i = 0; i < s->n_grid; ++i) {
        const double admitted = delta < s->grid[i] ? (double)miss_count : 0.0;
        volatile double a = s->decay * s->ema[i];
        volatile double b = omd * admitted;
        s->ema[i] = a + b;
    }
    if (++s->steps % s->period == 0) {
        int rc = bm_derive_beta(s->budget_bytes, s->expert_bytes, s->grid, s->ema, s->n_grid, s->beta, &s->beta);
        if (rc != BM_OK) return rc;
    }
    if (beta_out) *beta_out = s->beta;
    return BM_OK;
}
