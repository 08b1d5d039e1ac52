python -m paper_2509_12211_b200._build --force > /dev/null 2>&1 || exit 1
for c in ${CONFIGS:-c2 c3 c5}; do TS_PIPE_VERBOSE=1 timeout 120 python scripts/pipe_stamps.py $c 2>&1 | grep -v Warn | awk '!/pipe plan/ || !seen[$0]++' | head -24; done
