mkdir -p gpurun_out
bash tools/ablibs.sh "cur lu0 lu1" "f64:10" 1
