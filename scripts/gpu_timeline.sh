#!/bin/bash
# per-CTA render timeline of config 3 (experiments build, on the box only)
tag=${1:-t}
mkdir -p gpurun_out
python -m paper_2511_22793_b200.build --experiments > gpurun_out/timeline_build_$tag.log 2>&1
timeout 300 python scripts/timeline_c3.py > gpurun_out/timeline_c3_$tag.txt 2>&1
echo "rc=$?" >> gpurun_out/timeline_c3_$tag.txt
