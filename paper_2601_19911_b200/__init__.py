"""paper_2601_19911_b200: B200-native offload path for the `golp` OLAP engine
(arXiv 2601.19911, "GPU-Augmented OLAP Execution Engine: GPU Offloading").

Drop-in for the reference's device protocol (pkg/src/golp/device.py): a
`B200Device` ("b200" backend) whose topk()/probe() run hand-written sm_100a
kernels from libgolp_b200.so, with the reference's result layout, byte
accounting, ledgers, cost model and Risky Gate entry points kept under the same
names. Torch-tensor entry points for device-resident inputs live in
`paper_2601_19911_b200.resident`; multi-GPU sharding in `.sharded`.
"""

from .device import (
    BACKENDS,
    DEFAULT_MODELED_PROFILE,
    FULL_ROW,
    KEY_ONLY,
    MODES,
    OP_PROBE,
    OP_TOPK,
    B200Device,
    CostEstimate,
    DeviceCallResult,
    DeviceProfile,
    ModeledDevice,
    TransferLedger,
    calibrate_profile,
    device_probe,
    device_topk,
    estimate_device_cost,
    make_device,
    transfer_entry_bytes,
)
from .errors import (
    CalibrationError,
    CapacityError,
    GolpError,
    NoCrossingError,
    StrategyMismatchError,
    SweepBracketError,
)
from .gate import (
    DEFAULT_CPU_MODEL,
    DEVICE,
    HOST,
    OP_FULL_SORT,
    CpuCostModel,
    GateConfig,
    GateDecision,
    calibrate_cpu_model,
    decide,
    estimate_cpu_cost,
    execute_gated,
    execute_path,
    with_margin,
)
from .host import (
    KeyHashTable,
    ProbeResult,
    TopKResult,
    host_full_sort,
    host_hash_build,
    host_hash_probe,
    host_topk,
    key_bits,
    mix64,
    mix64_array,
)
from .store import (
    DEFAULT_PAYLOAD_BYTES,
    KEY_ENTRY_BYTES,
    ColumnTable,
    KeyVector,
    MaterializedJoin,
    MaterializedResult,
    extract_keys,
    full_row_bytes,
    generate_table,
    key_only_bytes,
    load_table,
    materialize,
    materialize_join,
    random_key_vector,
    random_keys,
    save_table,
)

__version__ = "0.1.0"
