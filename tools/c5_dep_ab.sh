# C5 deposit kernel A/B: launch list per library variant (tags as in tools/build_variants.sh; "main" = in-tree build)
for t in "$@"; do
  if [ "$t" = main ]; then unset PRNG_B200_LIB; else export PRNG_B200_LIB=$PWD/build/var_$t/libprng_b200.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l_$t.csv python bench.py --workload c5_full --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
  echo "== $t"; python tools/launch_share.py /tmp/l_$t.csv | grep calo_deposit
done
