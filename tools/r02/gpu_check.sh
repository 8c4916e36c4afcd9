#!/bin/bash
# Round-2 GPU check of a change: selected GPU tests (args) or the whole GPU suite.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-check}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout ${TMO:-1500} python -m pytest ${@:-tests -m gpu} -q -p no:cacheprovider --timeout 400 -x -rs > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -25 $O/pytest.log
