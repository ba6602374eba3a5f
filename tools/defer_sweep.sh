# deferred emission (RPQ_TUNE_DEFER) across configs
for d in ${DEFERS:-0 2 4}; do echo "defer $d"; EXTRA="--defer $d" CONFIGS="${CONFIGS:-cfg2 cfg3 cfg4 cfg5}" STEPS=8 bash tools/quick_bench.sh | cut -c1-60; done
