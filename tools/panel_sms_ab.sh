#!/bin/bash
# SMs left to the POTRF panel stream (MVN_POTRF_PANEL_SMS, read once per process) with the default
# super-panel width, alternating on one box.
for rep in 1 2; do
  for s in 4 6 8 2; do MVN_POTRF_PANEL_SMS=$s timeout 600 python tools/potrf_time.py D 2>&1 | tail -1 | sed "s/^/rep=$rep sms=$s /"; done
done
