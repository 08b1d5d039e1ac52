set -u
for v in "" "-DTS_EXP_F8_NOKCVT" "-DTS_EXP_F8_NOLO"; do
  TS_NVCC_EXTRA="$v" python -m paper_2509_12211_b200._build --force > /dev/null 2>&1 || exit 1
  echo "== $v"; timeout 300 python scripts/dense_fp8_time.py c3 2>&1 | grep dense
done
