"""Untrained corrective network and its optimiser (reference network.py),
GPU underneath: forward_net -> pdf_net_forward, grad_loss -> pdf_grad_loss,
adam_step -> pdf_adam_step."""
from .api import (AdamState, NetworkParams, adam_step, flatten_params, forward_net, grad_loss,  # noqa: F401
                  init_network, unflatten_params)
