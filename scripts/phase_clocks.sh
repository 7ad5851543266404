#!/bin/bash
# Per-phase SM cycles of the search (measurement build with -DVP_PHASE_CLOCKS, swapped in for the run).
#   bash scripts/phase_clocks.sh [profile_step args]   (on the GPU box; the .so is built here first:
#   nvcc ... -DVP_PHASE_CLOCKS -o phase_libvpb200.so)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
cp paper_2510_27191_b200/libvpb200.so /tmp/keep_libvpb200.so
cp phase_libvpb200.so paper_2510_27191_b200/libvpb200.so
python scripts/phase_clocks.py "$@"
cp /tmp/keep_libvpb200.so paper_2510_27191_b200/libvpb200.so
