# Virtual bf16/fp32 reduce-scatter (chunk-flag reduction path) under the
# current virtual-mode defaults, and worker-width / chunk / CTA variants.
set -x
for dt in bfloat16 float32; do
  python tools/virtual_rs_roofline.py --mib 64 --dtype $dt 2>&1 | tail -1
  for o in "worker_warps=2" "worker_warps=4" "worker_warps=8" "chunk_max=65536" "chunk_max=262144" "worker_warps=2 --opt chunk_max=262144" "worker_warps=4 --opt chunk_max=262144" "items_per_worker=2"; do
    python tools/virtual_rs_roofline.py --mib 64 --dtype $dt --opt $o 2>&1 | tail -1
  done
done
