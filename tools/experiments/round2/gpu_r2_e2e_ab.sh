# same-box A/B of the host-path chunk schedule (e2e_probe with two libraries)
for rep in 1 2; do
for v in old new; do
  for n in 10000 50000; do
    echo "== $v $n rep$rep"; SWR_LIB=tools/var/$v.so timeout -s KILL 600 python tools/e2e_probe.py $n 2>&1 | grep -E "chunk 256|1024:|copy_chunk  256"
  done
done
done
