for v in def p8 p8lb3 p12lb3; do
  if [ $v = def ]; then unset SPMV_LIB_PATH; else export SPMV_LIB_PATH=exp/$v/libspmv.so; fi
  timeout 600 python tools/exp_parts.py --config 4 --variants auto --parts all,long > gpurun_out/x_parts_$v.txt 2>&1
done
