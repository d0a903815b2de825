#!/bin/bash
# Dev sweep: kt_apply_host strategy x chunk size (elements) on pinned buffers.
for m in 0 2 1; do
  for c in 0 262144 524288 1048576 4194304; do
    if [ "$c" = 0 ]; then unset KT_HOST_CHUNK; else export KT_HOST_CHUNK=$c; fi
    echo "== mode $m chunk ${c:-default}"
    KT_HOST_ZEROCOPY=$m python tools/e2e_zc.py 2>&1 | grep -E "2\^24|2\^26"
    [ "$m" = 1 ] && break
  done
done
