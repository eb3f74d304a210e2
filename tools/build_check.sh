#!/bin/bash
# Build libfmap_cuda and fail loudly (used before every GPU run).
cd "$(dirname "$0")/.." && python -m paper_2604_10377_b200.build -v > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head; echo BUILD FAILED; exit 1; }
grep -E "spill" /tmp/build.log | sort | uniq -c | head -4
echo "built $(date +%T)"
