// fusegraph_b200_shim.hpp — the one addition the drop-in makes to the
// reference's API surface.  The shim keeps device mirrors of the stores and
// indexes it has seen, keyed in O(1) (table buffers + a 64-node sample
// checksum).  insert_batch / mark_delete (update.hpp:33-38), the reference's
// only sanctioned mutations of a built index (index.hpp:33), update the
// mirrors in place.  Code that edits a DocumentStore / HybridIndex's fields
// directly calls invalidate_device_mirrors() afterwards.
#pragma once

namespace fusegraph::b200 {
void invalidate_device_mirrors();
}
