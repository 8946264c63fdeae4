# Time the GPU worker (lib/paes_gpu_worker, the reference's __worker protocol) on a 4 GiB chunk and a
# 16-byte one (startup floor), and the reference parent's concatenation cost (cat of the part file).
set -e
python - <<'PY'
import numpy as np
np.random.default_rng(1).integers(0,256,(4<<30)+7,dtype=np.uint8).tofile('/dev/shm/wp_in.bin')
open('/dev/shm/wp_key','wb').write(bytes(range(16)))
PY
W=paper_1403_7295_b200/lib/paes_gpu_worker
N=$(( (4<<30) + 7 ))
export PAES_WORKER_TRACE=1
for i in 1 2 3; do
  s=$(date +%s.%N); $W __worker --in /dev/shm/wp_in.bin --offset 0 --len $N --final 1 --dir encrypt --keyfd 0 --out /dev/shm/wp.w0.1.part < /dev/shm/wp_key; e=$(date +%s.%N)
  echo "worker 4GiB: $(python -c "print(round($e-$s,3))") s"
done
s=$(date +%s.%N); $W __worker --in /dev/shm/wp_key --offset 0 --len 16 --final 1 --dir encrypt --keyfd 0 --out /dev/shm/wq.w0.1.part < /dev/shm/wp_key; e=$(date +%s.%N)
echo "worker 16B (startup floor): $(python -c "print(round($e-$s,3))") s"
s=$(date +%s.%N); cat /dev/shm/wp.w0.1.part > /dev/shm/wp_cat.bin; e=$(date +%s.%N)
echo "cat 4GiB part into fresh file: $(python -c "print(round($e-$s,3))") s"
rm -f /dev/shm/wp*
