for v in libdso_b200.so libdso_b200_d4.so libdso_b200_l4.so libdso_b200_bk8.so libdso_b200_all.so; do
  echo "$v $(DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout -s KILL 200 python scripts/c5_probe.py 2>&1 | grep 'train_tc=1')"
done
