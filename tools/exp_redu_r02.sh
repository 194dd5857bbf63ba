# A/B of bulk_reduce's vectors-per-lane on the virtual chunk-flag
# reduce-scatter; prebuilt variants in tools/bin/var/*.so (first run: u1/u2/u4
# for all types; second run: b1/b2 = 2-byte types at 1 or 2 vectors after the
# word-wise bf16 unpack).
L=paper_2402_06787_b200/lib/libforestcoll.so
cp $L /tmp/orig.so
for rep in 1 2; do
  for V in $(ls tools/bin/var/); do
    cp tools/bin/var/$V $L
    for dt in ${DTYPES:-bfloat16 float32}; do
      echo "$V rep=$rep $(python tools/virtual_rs_roofline.py --mib 64 --dtype $dt 2>&1 | tail -1)"
    done
  done
done
cp /tmp/orig.so $L
