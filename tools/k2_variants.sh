#!/bin/bash
# A/B of K2 build variants (paper_2509_18344_b200/_variants/lib_<name>.so): draft-pass time and the
# per-group sweep, alternating, each variant in its own process
mkdir -p gpurun_out
tag=${1:-kv}; shift
for rep in 1 2; do
  for v in default "$@"; do
    lib=paper_2509_18344_b200/libsubspec.so
    [ "$v" != default ] && lib=paper_2509_18344_b200/_variants/lib_$v.so
    echo -n "$v " >> gpurun_out/${tag}_variants.log
    SS_LIBSUBSPEC=$lib timeout 300 python tools/pass_time.py 6 2>&1 | tail -1 >> gpurun_out/${tag}_variants.log
  done
done
