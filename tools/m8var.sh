run() { echo "== $*"; env "$@" timeout 300 python bench.py --configs cfg4:m8 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read())
c=d['configs']['cfg4:m8']; print(c['value'], c['roofline']['frac'], c['roofline']['launch_us'])"; }
run TB_M8_GLUE_FIN=1
run TB_M8_GLUE_FIN=0
run TB_M8_GLUE_FIN=1
run TB_M8_GLUE_FIN=0
