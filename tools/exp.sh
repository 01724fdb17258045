for v in def u8 lb4 u8lb4 rg4 rg3; do
  if [ $v = def ]; then unset SPMV_LIB_PATH; else export SPMV_LIB_PATH=exp/$v/libspmv.so; fi
  timeout 600 python tools/exp_parts.py --config 4 --variants split --parts all,long > gpurun_out/x_parts_$v.txt 2>&1
done
unset SPMV_LIB_PATH
timeout 900 python -m pytest tests -m gpu -x -q -k "split or long or configs_full" > gpurun_out/x_pytest.txt 2>&1
