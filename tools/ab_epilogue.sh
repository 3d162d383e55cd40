# A/B of the CTA-pair GEMM's fused SwiGLU epilogues: the GEMM kernel tests on the
# current library, then the solo table rows of the fused nodes at TP=8 / TP=1 for a
# baseline library (exp_old/) and the current one, interleaved; then per-phase traces
# (exp_trace/, built with -DDH_GEMM_TRACE).
set +e
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" > gpurun_out/r02s3_gemm_tests.log 2>&1; tail -2 gpurun_out/r02s3_gemm_tests.log
for r in 1 2; do for lib in exp_old/libdh_b200.so paper_2411_15871_b200/lib/libdh_b200.so; do for tp in 8 1; do
  echo "== $lib tp=$tp round $r"; DH_LIB_PATH=$PWD/$lib timeout 300 python tools/solo_table.py --tp $tp --cap 132 | grep -E "mlp_up |mlp_down_dgrad|mlp_gate |mlp_gate_dgrad|total"
done; done; done
if [ -f exp_trace/libdh_b200.so ]; then
  for e in fwd bwd; do for shp in "4096 1792 4096 256 0 0" "4096 14336 4096 256 0 0"; do
    echo "== trace $shp EPI=$e"; DH_LIB_PATH=$PWD/exp_trace/libdh_b200.so EPI=$e timeout 60 python tools/gemm_trace.py $shp
  done; done
fi
