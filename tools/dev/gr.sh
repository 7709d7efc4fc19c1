#!/bin/bash
# gpurun from the repo root (so gpurun_out/ merges into /root/repo/gpurun_out)
cd /root/repo && rm -rf paper_2504_05638_b200/csrc/gpurun_out && exec /usr/local/graft/bin/gpurun "$@"
