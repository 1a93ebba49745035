/* Plain-C client of libdaso.so (no torch, no CUDA headers): exercises the host-only part
 * of the C ABI — schedule, plateau detector, LR schedule, layout helpers, init argument
 * validation — and prints the schedule records as CSV for the Python test to compare with
 * the oracle.  Built and run by tests/test_c_client.py. */
#include <stdio.h>
#include <string.h>

#include "daso.h"

#define CHECK(cond)                                                      \
    do {                                                                 \
        if (!(cond)) {                                                   \
            fprintf(stderr, "check failed: %s (line %d)\n", #cond, __LINE__); \
            return 1;                                                    \
        }                                                                \
    } while (0)

int main(void) {
    /* config 1 schedule: B=4, S=1, 2 GPUs per node, 20 steps */
    daso_sched_config sc = {4, 1, 1, 1, 5, 8, 2};
    daso_sched* s = NULL;
    CHECK(daso_sched_create(&sc, &s) == DASO_OK);
    for (int k = 0; k < 40; ++k) {
        daso_record r;
        const int plateau = (k == 16 || k == 24) ? 1 : 0;
        CHECK(daso_sched_next(s, plateau, &r) == DASO_OK);
        printf("%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld\n", (long long)r.step,
               (long long)r.phase, (long long)r.B, (long long)r.S, (long long)r.batch_in_cycle, (long long)r.send,
               (long long)r.blocking, (long long)r.send_group, (long long)r.merge, (long long)r.merge_S,
               (long long)r.merge_group, (long long)r.pending, (long long)r.due);
    }
    CHECK(daso_sched_destroy(s) == DASO_OK);

    daso_sched_config bad = {4, 5, 0, 0, 1, 8, 1}; /* S > B */
    CHECK(daso_sched_create(&bad, &s) == DASO_ERR_CONFIG);

    daso_plateau* p = NULL;
    int fired = 0, count = 0;
    CHECK(daso_plateau_create(5, 0.01, &p) == DASO_OK);
    for (int e = 0; e < 11; ++e) {
        CHECK(daso_plateau_update(p, 1.0, &fired) == DASO_OK);
        count += fired;
    }
    CHECK(count == 2);
    CHECK(daso_plateau_destroy(p) == DASO_OK);

    double lr = 0;
    CHECK(daso_lr_at(49, 10, 0.1, 4, 5, 0.5, 0, &lr) == DASO_OK && lr > 0.39999 && lr < 0.40001);

    size_t numel[3] = {3, 64, 65}, offs[3], total = 0;
    CHECK(daso_flat_layout(numel, 3, 64, offs, &total) == DASO_OK && offs[2] == 128 && total == 256);
    CHECK(daso_padded_numel(25557032, 4) == 25557248);

    daso_config cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.rank = 9;
    cfg.total_epochs = 1;
    cfg.steps_per_epoch = 64;
    daso_ctx* c = NULL;
    unsigned char uid[128] = {0};
    CHECK(daso_init(&c, 8, 4, 4, 1, &cfg, uid) == DASO_ERR_RANGE);
    cfg.rank = 0;
    CHECK(daso_init(&c, 8, 3, 4, 1, &cfg, uid) == DASO_ERR_CONFIG);
    CHECK(strcmp(daso_status_string(DASO_ERR_PROTOCOL), "protocol error") == 0);
    return 0;
}
