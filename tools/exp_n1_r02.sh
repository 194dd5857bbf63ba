# N=1 headline (nvs8 virtual allgather, 64 MiB shards): chunk size and worker width
for ch in 98304 131072 163840; do for w in 1 2; do for rep in 1 2; do
echo -n "chunk=$ch ww=$w: "
python tools/probe_virtual.py --coll allgather --mib 64 --opt chunk_max=$ch --opt worker_warps=$w 2>&1 | grep -o "algbw *[0-9.]* GB/s"
done; done; done
