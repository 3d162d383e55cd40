# A/B of a CTA-pair GEMM epilogue change: the GEMM kernel tests on the current
# library, then solo-table rows at TP=8 / TP=1 for a baseline library (exp_old/)
# and the current one, interleaved; then per-phase traces (exp_trace/, built with
# -DDH_GEMM_TRACE). ROWS: regex of solo-table rows; TRACES: "m n k pbn b_mn" list.
set +e
ROWS=${ROWS:-"mlp_up |mlp_down_dgrad|mlp_gate |mlp_gate_dgrad|total"}
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" > gpurun_out/ab_gemm_tests.log 2>&1; tail -2 gpurun_out/ab_gemm_tests.log
for r in 1 2; do for lib in exp_old/libdh_b200.so paper_2411_15871_b200/lib/libdh_b200.so; do for tp in 8 1; do
  echo "== $lib tp=$tp round $r"; DH_LIB_PATH=$PWD/$lib timeout 300 python tools/solo_table.py --tp $tp --cap 132 | grep -E "$ROWS"
done; done; done
if [ -f exp_trace/libdh_b200.so ]; then
  while read -r shp; do [ -z "$shp" ] && continue
    echo "== trace $shp EPI=${EPI:-}"; DH_LIB_PATH=$PWD/exp_trace/libdh_b200.so timeout 60 python tools/gemm_trace.py $shp 0
  done <<< "${TRACES:-}"
fi
