#!/bin/bash
# e2e copy/compute timeline of the host-buffer nest (N=32768, p=2): NNB_TRACE marks
cd "$(dirname "$0")/.."
NNB_DEBUG=1 NNB_TRACE=1 python tools/e2e_timeline.py "$@"
