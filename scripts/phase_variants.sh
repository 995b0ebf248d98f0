# per-role cycle breakdown (scripts/tc_phase.py) of phase-timing variant builds
# (scripts/build_variant.sh NAME "-DDSO_PHASE_TIMING ...")
OUT=gpurun_out/${1:-ph}; mkdir -p $OUT; shift
for v in "$@"; do
  echo "== $v" >> $OUT/phase.txt
  TC_PHASE_MODES=pipeline_csr DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/libdso_b200_$v.so timeout 300 python scripts/tc_phase.py >> $OUT/phase.txt 2>&1
done
