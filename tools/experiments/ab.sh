#!/bin/bash
# A/B two builds of libtlb200.so (build/ab/libA.so, libB.so), interleaved:
#   tools/experiments/ab.sh "<command printing one line>" [rounds]
cmd=$1; n=${2:-2}
for r in $(seq $n); do for v in A B; do echo -n "$v: "; TL_LIB=build/ab/lib$v.so bash -c "$cmd"; done; done
