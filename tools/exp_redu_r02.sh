# A/B of bulk_reduce's vectors-per-lane (FC_RED_U) on the virtual chunk-flag
# reduce-scatter / allreduce; prebuilt variants in tools/bin/var/u{1,2,4}.so.
L=paper_2402_06787_b200/lib/libforestcoll.so
cp $L /tmp/orig.so
for rep in 1 2; do
  for U in 1 2 4; do
    cp tools/bin/var/u$U.so $L
    for dt in bfloat16 float32; do
      echo "U=$U rep=$rep $(python tools/virtual_rs_roofline.py --mib 64 --dtype $dt 2>&1 | tail -1)"
    done
  done
done
cp /tmp/orig.so $L
