#!/bin/bash
# Round-2 GPU check of a change: selected GPU tests (args; KEXPR = pytest -k expression)
# or the whole GPU suite.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02/${TAG:-check}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -n "$KEXPR" ]; then
  timeout ${TMO:-1500} python -m pytest ${@:-tests -m gpu} -k "$KEXPR" -q -p no:cacheprovider --timeout 400 -rs > $O/pytest.log 2>&1
else
  timeout ${TMO:-1500} python -m pytest ${@:-tests -m gpu} -q -p no:cacheprovider --timeout 400 -rs > $O/pytest.log 2>&1
fi
echo "pytest rc=$?"; tail -25 $O/pytest.log
