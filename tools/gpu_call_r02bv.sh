#!/bin/bash
# final HEAD: full GPU suite on 4 GPUs (multi-GPU and 8-rank ring tests included)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bv_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/bv_pytest.log
