# A/B: bench lines for the current build under several env settings and for saved builds
# usage: bash scripts/r02_ab.sh "ENV=.. ENV2=.." ... ; libs in AB_LIBS
summ() { python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', round(d['value'],1), 'comp', round(r['compress_ms'],4), 'dec', round(r['decompress_ms'],4), 'step', round(d['ms_per_step'],4))"; }
W=${AB_WORKLOAD:-cfg2}
for L in ${AB_LIBS:-}; do FALCON_B200_LIB=$PWD/$L python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null | summ "lib=$L"; done
for E in "$@"; do env $E python bench.py --workload $W --steps 20 --warmup 3 --no-e2e --no-cpu 2>/dev/null | summ "$E"; done
