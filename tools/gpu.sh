#!/bin/bash
# usage: tools/gpu.sh <timeout_s> '<command>'   -- runs on the B200 box via gpurun
cd /root/repo || exit 1
T=${1:-900}; shift
timeout $((T + 1500)) /usr/local/graft/bin/gpurun --timeout "$T" -- "$@" > gpurun_out/last_call.log 2>&1
rc=$?
tail -3 gpurun_out/last_call.log
exit $rc
