#!/bin/bash
# full GPU suite, then the GPU suite under SLQ_GUARD=1, then smoke()
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_full.log 2>&1; echo "gpu suite rc $?"; tail -2 gpurun_out/gputests_full.log
SLQ_GUARD=1 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_guard.log 2>&1; echo "guard suite rc $?"; tail -2 gpurun_out/gputests_guard.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
