#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe/poison_run.py tok 2>&1 | tail -12
timeout 300 python tools/probe/poison_run.py bf16 2>&1 | tail -12
