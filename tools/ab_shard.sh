#!/bin/bash
# Per-shard timing (tools/probe_shard.py) for several library builds.
for lib in "$@"; do echo "== $lib"; GPP_B200_LIB=$lib python tools/probe_shard.py 2>&1 | cut -c1-80; done
