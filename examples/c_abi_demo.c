/* The C ABI from plain C (no C++, no torch): one agent's blocks offloaded while it "waits on a function call", then
 * uploaded into fresh blocks with the block table rewritten.  Runs on a metadata-only pool (device = -1: allocator,
 * tables and handles without KV bytes) unless a CUDA device ordinal is given as argv[1].
 *
 *   gcc -std=c11 -I include examples/c_abi_demo.c -L paper_2510_18586_b200 -ltokencake \
 *       -Wl,-rpath,paper_2510_18586_b200 -o /tmp/c_abi_demo && /tmp/c_abi_demo [device]
 */
#include <stdio.h>
#include <stdlib.h>

#include "tokencake.h"

#define CHECK(x)                                                                                  \
    do {                                                                                          \
        tc_status st_ = (x);                                                                      \
        if (st_ != TC_OK) {                                                                       \
            fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, tc_strerror(st_));        \
            return 1;                                                                             \
        }                                                                                         \
    } while (0)

int main(int argc, char **argv) {
    tc_pool_desc d;
    tc_pool_desc_init(&d, 28, 4, 128, 16, TC_BF16, 1024);   /* Qwen2.5-7B-shaped KV, 1024 blocks */
    d.device = argc > 1 ? atoi(argv[1]) : -1;
    d.host_slots = 256;
    tc_pool *p = NULL;
    CHECK(tc_pool_create_ex(&d, &p));
    if (d.device >= 0) CHECK(tc_fill_kv(p, 7));

    CHECK(tc_partition_reserve(p, 0, 64));                  /* a1: the critical class keeps 64 blocks */
    CHECK(tc_agent_add(p, 1, 0));
    int32_t ids[48], new_ids[48], table[48];
    CHECK(tc_alloc(p, 1, 48, ids));                         /* the agent's prompt + decode blocks */

    tc_handle h = 0;
    CHECK(tc_offload(p, 1, ids, 48, &h));                   /* a2-a4: the call starts; blocks go to the host */
    int64_t n = 0;
    CHECK(tc_block_table(p, 1, table, 48, &n));
    if (n != 48 || table[0] != -1) { fprintf(stderr, "table not marked host-resident\n"); return 1; }
    CHECK(tc_sync(p));                                      /* the source blocks retire */

    CHECK(tc_upload(p, h, new_ids));                        /* a5-a7: before the call returns */
    CHECK(tc_wait(p, h));
    CHECK(tc_block_table(p, 1, table, 48, &n));
    for (int i = 0; i < 48; ++i)
        if (table[i] != new_ids[i]) { fprintf(stderr, "remap mismatch at %d\n", i); return 1; }
    tc_stats_t s;
    CHECK(tc_stats(p, &s));
    printf("ok: 48 blocks offloaded and uploaded; first new id %d; free %lld alloc %lld host_free %lld\n",
           new_ids[0], (long long)s.free_blocks, (long long)s.alloc_blocks, (long long)s.host_free);

    /* the asynchronous serving loop: each cycle offloads the agent and uploads it back, and retires with
       a lag of 2 (reading A8''): the last two cycles' transfers keep streaming while the next one is enqueued */
    for (int c = 0; c < 6; ++c) {
        CHECK(tc_block_table(p, 1, table, 48, &n));
        CHECK(tc_offload(p, 1, table, 48, &h));
        CHECK(tc_upload(p, h, new_ids));
        CHECK(tc_retire_lag(p, 2));
    }
    if (tc_retire_lag(p, 0) != TC_E_INVAL) { fprintf(stderr, "lag 0 not refused\n"); return 1; }
    CHECK(tc_sync(p));
    CHECK(tc_stats(p, &s));
    if (s.free_blocks + s.alloc_blocks != 1024 || s.alloc_blocks != 48 || s.host_free != 256) {
        fprintf(stderr, "counters after the loop: free %lld alloc %lld host_free %lld\n", (long long)s.free_blocks,
                (long long)s.alloc_blocks, (long long)s.host_free);
        return 1;
    }
    printf("ok: 6 retire-lag cycles; free %lld alloc %lld host_free %lld\n", (long long)s.free_blocks,
           (long long)s.alloc_blocks, (long long)s.host_free);
    tc_pool_destroy(p);
    return 0;
}
