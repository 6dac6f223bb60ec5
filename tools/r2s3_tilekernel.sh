set -u
mkdir -p gpurun_out
(FV2D_TILE_MAX_CELLS=1000000000000 timeout 1500 python -m pytest tests -m gpu -q -k "not spray and not source and not recon" > gpurun_out/s3x_pytest_tile.txt 2>&1; echo "exit $?" >> gpurun_out/s3x_pytest_tile.txt)
FV2D_TILE_MAX_CELLS=0 timeout 600 python tools/tile_bench.py > gpurun_out/s3x_pair.jsonl 2>&1
FV2D_TILE_MAX_CELLS=1000000000000 timeout 600 python tools/tile_bench.py > gpurun_out/s3x_tile.jsonl 2>&1
echo done
