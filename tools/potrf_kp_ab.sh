#!/bin/bash
# Super-panel width at D and E beyond kp = 4 (MVN_POTRF_KP, read once per process).
for rep in 1 2; do
  for kp in 4 8; do MVN_POTRF_KP=$kp timeout 600 python tools/potrf_time.py D 2>&1 | tail -1 | sed "s/^/rep=$rep kp=$kp /"; done
done
for kp in 6 8; do MVN_POTRF_KP=$kp timeout 900 python tools/potrf_time.py E 2>&1 | tail -1 | sed "s/^/kp=$kp /"; done
for kp in 3 6 8; do MVN_POTRF_KP=$kp timeout 600 python tools/potrf_time.py D 2 160 2>&1 | tail -1 | sed "s/^/kp=$kp /"; done
