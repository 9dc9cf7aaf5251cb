for v in base t2a t2b t2c t2d; do
  if [ $v = base ]; then unset TB_LIB; else export TB_LIB=tools/lib_$v.so; fi
  GRAPH=1 timeout 300 python tools/ncu_stack.py cfg2 tl2 1 32 > gpurun_out/v_$v.txt 2>&1
  echo "$v $(tail -n 1 gpurun_out/v_$v.txt)"
done
