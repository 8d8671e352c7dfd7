#!/bin/bash
cd $GRAFT_REPO_ROOT
P=r2g
timeout 1800 python -m pytest tests -q -m gpu --durations=30 > gpurun_out/${P}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${P}_tests.log
P=r2p bash profiles/scripts/r2_profile_c4.sh
