#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 180 build/gate_probe 2>&1 | grep -E "ks=|back-to-back" | sed -E 's/\| cta0.*scan cta:/| scan:/'
