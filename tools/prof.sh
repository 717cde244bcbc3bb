#!/bin/bash
# usage (on the GPU box): tools/prof.sh <name> <probe args...>
name=$1; shift
ncu --set full --import-source on --clock-control none -k regex:k_sssp -c 1 -o gpurun_out/$name python tools/probe.py "$@" > gpurun_out/$name.log 2>&1
