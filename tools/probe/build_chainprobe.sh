#!/bin/sh
# probe build of the library (-DPF_CHAIN_PROBE) for tools/probe/chain_probe.py
set -e
R=$(cd "$(dirname "$0")/../.." && pwd)
make -C "$R/paper_2211_14133_b200" OUT="$R/tools/probe/chainprobe" OBJ="$R/tools/probe/chainprobe/obj" \
     NVFLAGS_EXTRA=-DPF_CHAIN_PROBE "$R/tools/probe/chainprobe/libpf_b200.so"
