#!/bin/bash
# Same-box A/B of ab/base.so vs ab/new.so over several workloads (run via gpurun), alternating.
# Usage: bash tools/ab_multi.sh REPS "<bench args 1>" "<bench args 2>" ...
REPS=$1; shift
for args in "$@"; do echo "== $args"; bash tools/ab_lib.sh $REPS "$args"; done
