mkdir -p gpurun_out
for rep in 1 2 3; do
  TSW_LIB=$PWD/paper_2005_11931_b200/libtsw_variant.so timeout 120 python tools/abtest.py f64 4,5 3 2>&1 | sed 's/^/nocache /'
  timeout 120 python tools/abtest.py f64 4,5 3 2>&1 | sed 's/^/smem    /'
done
