timeout 1200 python tools/cusparse_context.py --configs 2,3,4,5 --out gpurun_out/x_cusparse.json > gpurun_out/x_cusparse.txt 2>&1
