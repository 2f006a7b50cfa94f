#!/bin/bash
cd "$GRAFT_REPO_ROOT"
bash gpurun_cycle.sh
bash gpurun_prof_all.sh
