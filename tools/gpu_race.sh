# race-perturbation test (compute-sanitizer is closed on this pool): the TB/energy/peer/parity
# suites against a build with random per-warp delays around every row barrier (TSW_TB_JITTER=1)
mkdir -p gpurun_out
for rep in 1 2; do
  TSW_LIB=abl/jit.so timeout 1200 python -m pytest tests/test_tblock_gpu.py tests/test_energy_fused_gpu.py tests/test_peer_gpu.py \
    tests/test_parity_gpu.py -q -p no:cacheprovider -k "not config3_full and not config4_full and not config5_batched" \
    > gpurun_out/race_jitter_$rep.log 2>&1
  echo "rep $rep rc=$? $(tail -1 gpurun_out/race_jitter_$rep.log)"
done
