#!/bin/bash
# Build and run the pair speed-of-light microbenchmark on one B200.
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o pair_sol pair_sol.cu
PAIRS=$(python -c "import json;d=json.load(open('pairs_c3.json'));print(d['included_pairs_per_step']/len(d['views']))" 2>/dev/null || echo 14.8e6)
./pair_sol "$PAIRS"
