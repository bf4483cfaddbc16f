#!/bin/bash
# C2 factorize+solve under different glibc malloc settings (host-bound engine:
# how much of the create time is allocator work).  Run on the GPU box.
cd "$(dirname "$0")/.."
run() {
    echo "== $1"
    shift
    env "$@" REPS=4 python tools/time_c2.py 512 2>&1 | grep -E "^n=512" | tail -3
}
run baseline X=1
run "mmap/trim thresholds 1G, top pad 256M" MALLOC_MMAP_THRESHOLD_=1073741824 MALLOC_TRIM_THRESHOLD_=4294967296 MALLOC_TOP_PAD_=268435456
run "tunables + tcache 1024" GLIBC_TUNABLES=glibc.malloc.mmap_threshold=1073741824:glibc.malloc.trim_threshold=4294967296:glibc.malloc.top_pad=268435456:glibc.malloc.tcache_count=1024
run "arena max 1" MALLOC_ARENA_MAX=1
