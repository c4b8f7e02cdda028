#!/bin/bash
# compute-sanitizer over the async-copy / shared-memory kernels (passes A/B/C of the
# partitioned path, k-mer front end, string kernel, single-key kernels) at test sizes.
#   bash tools/sanitize.sh memcheck|racecheck|synccheck   (one tool per GPU call)
TOOL=${1:-memcheck}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
SEL="test_partitioned_u64_vs_reference and (1 or 4097) or test_partitioned_skewed_streams_spill or test_partitioned_unaligned_buffers or test_partitioned_kmers_edges or test_partitioned_golden_fixtures or test_string_keys_vs_reference or test_golden_single_key or test_single_key"
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool "$TOOL" --error-exitcode 99 \
    --print-limit 50 --log-file "gpurun_out/sanitize_${TOOL}.log" \
    python -m pytest tests/test_gpu_partition.py tests/test_gpu_parity.py tests/test_gpu_host_api.py \
    -q -m gpu -p no:cacheprovider -k "$SEL" > "gpurun_out/sanitize_${TOOL}_pytest.txt" 2>&1
echo "sanitizer $TOOL rc=$?"
tail -3 "gpurun_out/sanitize_${TOOL}_pytest.txt"
tail -5 "gpurun_out/sanitize_${TOOL}.log"
