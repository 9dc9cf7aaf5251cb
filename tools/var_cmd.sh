for v in base noq nocomp notail rt56 rt56m3; do
  if [ $v = base ]; then unset TB_LIB; else export TB_LIB=tools/lib_$v.so; fi
  echo "== $v"; timeout 300 python tools/ncu_stack.py cfg4 i2s 1 16 2>&1 | tail -1
  timeout 300 python tools/ncu_stack.py cfg2 i2s 1 32 2>&1 | tail -1
done
