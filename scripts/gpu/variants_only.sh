# the k_lamb variants of build/variants only
mkdir -p gpurun_out
export SP_SKIP_BUILD=1
bash scripts/gpu/variants.sh
