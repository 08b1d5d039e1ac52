set -u
TS_NVCC_EXTRA="-DTS_EXP_R16" python -m paper_2509_12211_b200._build --dev --force > /dev/null 2>&1 || exit 1
b() { TS_DEV_LIB=1 env "$@" timeout 300 python bench.py --config $CFG --steps 400 --warmup 10 --no-dense --no-e2e --no-reuse --no-oracle --no-spread 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$CFG $*', round(j['ms_per_step']*1e3,2))"; }
CFG=c3; b X=1; b TS_SC_R=16; b TS_SC_R=16 TS_SC_CMAX=2; b TS_SC_R=16 TS_SC_CMAX=3
CFG=c5; b X=1; b TS_SC_R=16; b TS_SC_R=16 TS_SC_CMAX=9
CFG=c2; b X=1; b TS_SC_R=8
