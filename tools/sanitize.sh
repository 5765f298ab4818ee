#!/bin/bash
# compute-sanitizer passes over one small DFS tree step (the smoke case: SMALL model, 2 prompts x 4
# branches, __graft_entry__.smoke) on the GPU box:
#   memcheck  --leak-check full   (out-of-bounds / misaligned global + shared accesses, leaks)
#   racecheck (shared-memory hazards), with the default CTA-pair GEMMs and again with single-CTA GEMMs
#   (gemm_2cta 0): the CTA-pair run reports only the 8 reserved shared-memory bytes 0x58-0x5f that
#   tcgen05.alloc.cta_group::2 uses for its cross-CTA handshake (written before the kernel body).
# Logs: gpurun_out/sanitize_{memcheck,racecheck,racecheck_1cta}.log
set -u
O=gpurun_out
mkdir -p $O
S="import sys; sys.path.insert(0, '.'); import __graft_entry__ as g; g.smoke()"
S1="import sys; sys.path.insert(0, '.'); import __graft_entry__ as g; g.smoke({'gemm_2cta': 0})"
timeout 1200 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python -c "$S" > $O/sanitize_memcheck.log 2>&1
echo "memcheck rc=$?" >> $O/sanitize_memcheck.log
timeout 1800 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python -c "$S" > $O/sanitize_racecheck.log 2>&1
echo "racecheck rc=$?" >> $O/sanitize_racecheck.log
timeout 1800 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python -c "$S1" > $O/sanitize_racecheck_1cta.log 2>&1
echo "racecheck (gemm_2cta 0) rc=$?" >> $O/sanitize_racecheck_1cta.log
for f in memcheck racecheck racecheck_1cta; do tail -n 3 $O/sanitize_$f.log; done
