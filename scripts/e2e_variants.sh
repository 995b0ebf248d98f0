for v in ${VARIANTS:-libdso_b200.so}; do
  echo "$v $(DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-stages --no-extra 2>&1 | grep -o '"e2e": {"value": [0-9.e+]*' )"
done
