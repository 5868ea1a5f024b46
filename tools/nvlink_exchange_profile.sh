# NVLink bytes of the fused tensor-parallel exchange (needs >= 2 GPUs; run from the repo root):
#   bash tools/nvlink_exchange_profile.sh [world] [model]
# One rank of tools/tp_ipc_check.py runs under ncu (never wrap the whole multi-rank launch in ncu); the
# others run plainly.  Expected per forward and rank: ~2 * layers * hidden * rows * 4 B * (world - 1)
# sent (O and down partial tiles to every peer) + the LM-head (max, id) pairs.
W=${1:-2}; M=${2:-tiny-qwen}
mkdir -p gpurun_out
for r in $(seq 1 $((W - 1))); do
  RANK=$r WORLD_SIZE=$W MASTER_ADDR=127.0.0.1 MASTER_PORT=29911 DBL_TP_IPC_MODEL=$M \
    python tools/tp_ipc_check.py > gpurun_out/nvl_rank$r.txt 2>&1 &
done
RANK=0 WORLD_SIZE=$W MASTER_ADDR=127.0.0.1 MASTER_PORT=29911 DBL_TP_IPC_MODEL=$M \
  ncu --clock-control none -k regex:fwd_kernel -c 4 \
      --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum \
      --csv --log-file gpurun_out/nvl_exchange.csv python tools/tp_ipc_check.py > gpurun_out/nvl_rank0.txt 2>&1
wait
cat gpurun_out/nvl_exchange.csv | tail -20
