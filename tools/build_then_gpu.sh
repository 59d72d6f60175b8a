#!/bin/bash
# build locally (abort on failure), then run the given command on the GPU box
cd /root/repo
python -m paper_1409_7166_b200.build > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head; echo BUILD FAILED; exit 1; }
T=${GPU_TIMEOUT:-900}
timeout $((T + 1200)) /usr/local/graft/bin/gpurun --timeout $T -- "$@"
