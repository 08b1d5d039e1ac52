set -u
python -m paper_2509_12211_b200._build > /dev/null 2>&1 || exit 1
e() { env "$@" timeout 300 python bench.py --config $CFG --steps 600 --warmup 10 --no-dense --no-reuse --no-oracle --no-spread 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=j['e2e']; print('$CFG $*', 'dev', round(j['ms_per_step']*1e3,2), 'e2e', round(e['ms_per_step']*1e3,2), e['steps'])"; }
for CFG in c3 c2 c5 c4; do e X=1; e TS_E2E_NB=16; e TS_E2E_NOCOPY=1; done
