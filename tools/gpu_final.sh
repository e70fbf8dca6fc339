#!/usr/bin/env bash
# Full GPU test suite + smoke() on the GPU box (what the driver runs at round end).
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/tests.log 2>&1; echo tests=$?; tail -4 gpurun_out/final/tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke=$?; tail -3 gpurun_out/final/smoke.log
