# N=1 headline (nvs8 virtual allgather, 64 MiB shards): CTA count and chunk size
for c in 16 18; do for ch in 32768 65536 131072; do
echo -n "ctas=$c chunk=$ch: "
python tools/probe_virtual.py --coll allgather --mib 64 --opt ctas_per_rank=$c --opt chunk_max=$ch 2>&1 | grep -o "algbw *[0-9.]* GB/s"
done; done
echo -n "configs0 8x1MiB default: "; python tools/probe_virtual.py --coll allgather --mib 1 2>&1 | grep -o "algbw *[0-9.]* GB/s"
echo -n "configs0 8x1MiB chunk 64K: "; python tools/probe_virtual.py --coll allgather --mib 1 --opt chunk_max=65536 2>&1 | grep -o "algbw *[0-9.]* GB/s"
