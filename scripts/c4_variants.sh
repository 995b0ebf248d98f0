for v in ${VARIANTS:-libdso_b200.so}; do
  echo "$v $(DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout -s KILL 200 python scripts/c4_time.py 2>&1 | tail -1)"
done
